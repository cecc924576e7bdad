import sys, os, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_09584_b200 import _capi
lib = _capi.load()
t, ms = C.c_double(), C.c_double()
_capi.check(lib.bp_measure_fp32_peak(0, C.byref(t), C.byref(ms)))
print(f"fp32 ffma peak {t.value:.1f} TFLOP/s ({ms.value:.2f} ms)")
lib.bp_measure_fp32_peak_reg.restype = C.c_int
lib.bp_measure_fp32_peak_reg.argtypes = [C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double)]
_capi.check(lib.bp_measure_fp32_peak_reg(0, C.byref(t), C.byref(ms)))
print(f"fp32 ffma 3-register (acc += x*w) {t.value:.1f} TFLOP/s ({ms.value:.2f} ms)")
