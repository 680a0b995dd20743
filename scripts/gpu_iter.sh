# one build -> measure iteration: parity tests, bench line, launch lists, ncu --set full of the kernels
# usage: bash scripts/gpu_iter.sh TAG
TAG=${1:-it}
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -x -q -m gpu 2>&1 | tail -15
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; tail -3 gpurun_out/bench_$TAG.err
cat gpurun_out/bench_$TAG.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python scripts/profile_infer.py 10000 > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_train_$TAG.csv python scripts/profile_infer.py 1000 --train > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_hidden|k_output|k_gsum" -s 6 -c 3 -o gpurun_out/prof_$TAG python scripts/profile_infer.py 10000 > gpurun_out/ncu_$TAG.log 2>&1; tail -3 gpurun_out/ncu_$TAG.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_normad_cl|k_shard|k_compact" -s 3 -c 3 -o gpurun_out/prof_train_$TAG python scripts/profile_infer.py 300 --train > gpurun_out/ncu_train_$TAG.log 2>&1; tail -3 gpurun_out/ncu_train_$TAG.log
ls -la gpurun_out
