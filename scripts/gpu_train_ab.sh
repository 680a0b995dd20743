mkdir -p gpurun_out
timeout 300 python scripts/train_time.py 2>&1 | tail -3
timeout 1500 python -m pytest tests/ -q -x -m gpu -p no:cacheprovider > gpurun_out/tr_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/tr_pytest.log
