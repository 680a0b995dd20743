import ctypes, sys
sys.path.insert(0, "/root/repo")
from paper_1711_03637_b200.build import PEAKS_OUT
lib = ctypes.CDLL(PEAKS_OUT)
x = ctypes.c_double()
for _ in range(3):
    lib.snn_measure_dp_latency(ctypes.byref(x)); print("fp64 dependent add/mul latency (cycles):", x.value)
