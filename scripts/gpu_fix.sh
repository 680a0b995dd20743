timeout 300 python scripts/gb_ab.py 3 1 2>&1 | tail -2
for n in 1250 10000; do python scripts/infer_time.py $n; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fix_launches.csv python scripts/profile_infer.py 10000 > /dev/null 2>&1
grep k_hidden_fix gpurun_out/fix_launches.csv | tail -1 | awk -F'","' '{print $5, $NF}'
timeout 1500 python -m pytest tests/ -q -x -m gpu -p no:cacheprovider > gpurun_out/fix_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/fix_pytest.log
