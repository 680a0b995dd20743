mkdir -p gpurun_out
timeout 300 python scripts/gb_ab.py 3 1 2>&1 | tail -3
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/gb3_launches.csv python scripts/profile_infer.py 10000 > /dev/null 2>&1; echo "launches rc=$?"
grep -E "k_hidden" gpurun_out/gb3_launches.csv | tail -2 | cut -c1-200
timeout 900 python -m pytest tests/ -q -x -m gpu -p no:cacheprovider > gpurun_out/gb3_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/gb3_pytest.log
