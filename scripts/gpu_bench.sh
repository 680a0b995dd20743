mkdir -p gpurun_out
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_${1:-x}.json 2> gpurun_out/bench_${1:-x}.err; echo "bench rc=$?"
tail -3 gpurun_out/bench_${1:-x}.err
