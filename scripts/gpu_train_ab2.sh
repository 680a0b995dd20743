bash scripts/variants.sh scripts/train_time.py base scan base scan 2>&1 | grep -E "===|train:"
bash scripts/gpu_phases_ab.sh pscan 2>&1
cp variants/libscan.so paper_1711_03637_b200/libsnn_b200.so
timeout 1500 python -m pytest tests/ -q -x -m gpu -p no:cacheprovider -k "train or normad or c5 or epoch or toy or dt01 or shim or refsuite" > gpurun_out/tr2_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/tr2_pytest.log
