"""A/B of the two packed-BMM kernels (btnn_cuda_set_bmm_kernel): graph-replayed kernel time
of bmm_pm1 (-> int32) and bmm_pm1_bin (-> bits) at n x n x n, and the fraction of the measured
tcgen05 i8 peak. Usage: python scripts/bmm_kernels.py [n ...]"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_16578_b200 import capi  # noqa: E402

PEAK_OPS = 2 * 2282e12  # bit-ops/s: measured kind::i8 N=256 MAC rate x 2


def main():
    sizes = [int(v) for v in sys.argv[1:]] or [1024, 2048, 4096, 8192]
    lib = capi.lib()
    med, mn, kns = C.c_double(), C.c_double(), C.c_double()
    eng = C.create_string_buffer(24)
    rb = capi.BenchReadback(None, None, None, C.pointer(kns), None, None)
    for n in sizes:
        for bin_ in (0, 1):
            for which, name in ((capi.BMM_WHOLE_K, "whole"), (capi.BMM_PIPELINED, "pipe")):
                if which == capi.BMM_WHOLE_K and n > 1536:
                    continue
                capi.set_bmm_kernel(which)
                capi.check(lib.btnn_cuda_bench_bmm(n, bin_, 20, 5, C.byref(med), C.byref(mn), eng, 24, C.byref(rb)))
                ops = 2.0 * n ** 3
                print(f"n={n:5d} {'bin' if bin_ else 'i32'} {name:5s} kernel {kns.value / 1e3:9.2f} us  call {med.value / 1e3:9.2f} us"
                      f"  {ops / kns.value / 1e3:8.1f} T bit-op/s  frac {ops / (kns.value * 1e-9) / PEAK_OPS:.3f}"
                      f"  [{eng.value.decode()}]", flush=True)
    capi.set_bmm_kernel(capi.BMM_AUTO)


if __name__ == "__main__":
    main()
