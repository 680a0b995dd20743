# guard-band v2: A/B against v1 and float64, launch list, ncu capture, round-2 tests
mkdir -p gpurun_out
timeout 300 python scripts/gb_ab.py 3 4 1 2>&1 | tail -5
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/gb2_launches.csv python scripts/profile_infer.py 10000 > /dev/null 2>&1; echo "launches rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_hidden_gb|k_hidden_fix" -s 2 -c 2 -o gpurun_out/prof_gb2 python scripts/profile_infer.py 10000 > gpurun_out/ncu_gb2.log 2>&1; echo "ncu rc=$?"
timeout 900 python -m pytest tests/test_gpu_round2.py tests/test_gpu_parity.py -q -x -m gpu -p no:cacheprovider > gpurun_out/gb2_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/gb2_pytest.log
