# round 2: GPU tests (incl. the reference's own suite through the shim), then the bench
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests/ -q -m gpu -p no:cacheprovider --durations=15 > gpurun_out/r2_pytest.log 2>&1; echo "pytest rc=$?"
tail -40 gpurun_out/r2_pytest.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err; echo "bench rc=$?"
tail -5 gpurun_out/r2_bench.err
