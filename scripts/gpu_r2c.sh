# round 2 (re-entry): GPU tests with the guard-band hidden kernel, then the bench
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 600 python -m pytest tests/test_gpu_round2.py -q -x -m gpu -p no:cacheprovider -k guard_band -s > gpurun_out/r2c_gb.log 2>&1; echo "gb rc=$?"
tail -15 gpurun_out/r2c_gb.log
timeout 2400 python -m pytest tests/ -q -m gpu -p no:cacheprovider --durations=15 > gpurun_out/r2c_pytest.log 2>&1; echo "pytest rc=$?"
tail -40 gpurun_out/r2c_pytest.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r2c_bench.json 2> gpurun_out/r2c_bench.err; echo "bench rc=$?"
tail -5 gpurun_out/r2c_bench.err
