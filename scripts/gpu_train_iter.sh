# training iteration: training parity tests, bench (train + c5), ncu of the sequential kernel
TAG=${1:-tr}
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "train or c5 or zero_error or non_finite" 2>&1 | tail -15
timeout 900 python bench.py --steps 5 --warmup 3 --skip-latency > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; tail -3 gpurun_out/bench_$TAG.err
cat gpurun_out/bench_$TAG.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_train_$TAG.csv python scripts/profile_infer.py 1000 --train > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_normad|k_shard" -s 2 -c 2 -o gpurun_out/prof_train_$TAG python scripts/profile_infer.py 300 --train > gpurun_out/ncu_train_$TAG.log 2>&1; tail -3 gpurun_out/ncu_train_$TAG.log
