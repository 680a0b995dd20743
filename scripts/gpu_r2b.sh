# round 2: tests, bench, e2e breakdown, launch lists + ncu full captures (profiles/r02_*)
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/ -q -m gpu -p no:cacheprovider > gpurun_out/r2_pytest.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/r2_pytest.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
tail -3 gpurun_out/bench.err
timeout 300 python scripts/e2e_breakdown.py > gpurun_out/e2e_breakdown.txt 2>&1
cat gpurun_out/e2e_breakdown.txt
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python scripts/profile_infer.py 10000 > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_train.csv python scripts/profile_infer.py 1000 --train > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_prep|k_tile_scan|k_hidden|k_gsum|k_output" -s 10 -c 5 -o gpurun_out/prof_r2i python scripts/profile_infer.py 10000 > gpurun_out/ncu_infer.log 2>&1; tail -2 gpurun_out/ncu_infer.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_compact|k_shard|k_normad" -s 6 -c 3 -o gpurun_out/prof_r2t python scripts/profile_infer.py 300 --train > gpurun_out/ncu_train.log 2>&1; tail -2 gpurun_out/ncu_train.log
ls -la gpurun_out | tail -20
timeout 300 python scripts/train_phases.py > gpurun_out/train_phases.txt 2>&1; cat gpurun_out/train_phases.txt
