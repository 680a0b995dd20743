# parity tests, bench line, launch list, one full ncu capture of the hot kernel
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -x -q -m gpu 2>&1 | tail -15
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err
cat gpurun_out/bench.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python scripts/profile_infer.py 10000 > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_train.csv python scripts/profile_infer.py 1000 --train > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_hidden|k_output" -s 4 -c 2 -o gpurun_out/prof_infer python scripts/profile_infer.py 3000 > gpurun_out/ncu_infer.log 2>&1; tail -3 gpurun_out/ncu_infer.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_normad -s 2 -c 1 -o gpurun_out/prof_normad python scripts/profile_infer.py 300 --train > gpurun_out/ncu_normad.log 2>&1; tail -3 gpurun_out/ncu_normad.log
ls -la gpurun_out
