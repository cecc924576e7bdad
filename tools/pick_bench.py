"""Host pick_out + prune cost at multi-GPU scale (dev helper): bp_pick_out (host.cu pick_indices,
bab.cpp:85-153) on a pool of N records picking n (eta = 0.75, T = 0.05), vs the oracle's
restatement; prints ms per call.  python tools/pick_bench.py [N] [n]"""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2412_09584_b200 import _capi  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
n = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
lib = _capi.load()
rng = np.random.default_rng(0)
meta = (_capi.PoolMeta * N)()
lf = rng.normal(size=N) * 10
uf = lf + np.abs(rng.normal(size=N)) * 5
for i in range(N):
    meta[i] = _capi.PoolMeta(float(lf[i]), float(uf[i]), i + 1, float(-rng.uniform(0, 30)))
h = C.c_void_p()
_capi.check(lib.bp_rng_new(7, C.byref(h)))
picked = (C.c_int * n)()
k = C.c_int()
t0 = time.perf_counter()
reps = 3
for _ in range(reps):
    _capi.check(lib.bp_pick_out(meta, N, n, 0.75, 0.05, h, picked, C.byref(k)))
dt = (time.perf_counter() - t0) / reps
print(f"pick_out N={N} n={n}: {1e3 * dt:.1f} ms per call, picked {k.value}, first {list(picked)[:5]}")
