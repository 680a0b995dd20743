# ncu captures of the inference kernels + FP64 latency microbenchmark
set -x
mkdir -p gpurun_out
python -c "
import ctypes; from paper_1711_03637_b200.build import PEAKS_OUT
lib=ctypes.CDLL(PEAKS_OUT); c=ctypes.c_double(); lib.snn_measure_dp_latency(ctypes.byref(c)); print('dp_latency_cycles', c.value)
f64=ctypes.c_double(); f32=ctypes.c_double(); lib.snn_measure_fma_peaks(ctypes.byref(f64), ctypes.byref(f32)); print('peaks', f64.value, f32.value)
" | tee gpurun_out/dp_latency.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_hidden|k_output" -s 4 -c 2 -o gpurun_out/prof_infer2 python scripts/profile_infer.py 3000 > gpurun_out/ncu_infer2.log 2>&1; tail -3 gpurun_out/ncu_infer2.log
