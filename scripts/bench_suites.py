"""GPU rows for the reference's benchmark suites, in its CSV schema.

Mirrors `btnn bench --suite bmm|bmm-bin|bconv|bconv-bin|model --csv` (btnn_cli.cpp:113-130,
bench.hpp:129-378): same suites, shapes, seed line and columns
(suite,kernel,variant,layout,shape,threads,reps,warmup,median_ns,mean_ns,min_ns,throughput,
throughput_unit,precheck), with the B200 path timed through the C ABI:

* bmm / bmm-bin: n x n x n for n = 128 .. max (the paper's §7.2 sweep), bit-ops/s = 2 n^3 / t
  (bench.hpp:207-209); the general scheme times float binarization + BMM, the bin scheme packed
  operands + binarized output, as the reference does.
* bconv / bconv-bin: 64x64 input, batch 16, 3x3, C = O = 128 .. 2048 (§7.3 sweep), bit-ops/s =
  2 P Q N C O K^2 / t (bench.hpp:290-292).
* model: images/s of the device plan over --batches (graph replay, inputs resident).

`precheck` is a GPU-side cross-engine check (tcgen05 path vs the CUDA-core POPC path give the
same outputs / logits bit for bit); the CPU oracle stays in tests/.
Device-timed (CUDA events), median of `reps` after `warmup`.

  python scripts/bench_suites.py --suite bconv-bin --csv out.csv
"""
import argparse
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2006_16578_b200 import btnn, capi  # noqa: E402
from paper_2006_16578_b200 import model as M  # noqa: E402
from paper_2006_16578_b200 import weights as W  # noqa: E402

HDR = ("suite,kernel,variant,layout,shape,threads,reps,warmup,median_ns,mean_ns,min_ns,throughput,"
       "throughput_unit,precheck")


def row(suite, kernel, variant, shape, reps, warmup, med, mn, thr, unit, ok):
    return (f"{suite},{kernel},{variant},plain,{shape},0,{reps},{warmup},{med:.1f},{med:.1f},{mn:.1f},"
            f"{thr:.3f},{unit},{'ok' if ok else 'FAIL'}")


def bmm_rows(bin_, reps, warmup, nmin, nmax):
    lib = capi.lib()
    med, mn = C.c_double(), C.c_double()
    eng = C.create_string_buffer(16)
    out = []
    n = nmin
    while n <= nmax:
        capi.check(lib.btnn_cuda_bench_bmm(n, int(bin_), reps, warmup, C.byref(med), C.byref(mn), eng, 16))
        ops = 2.0 * n ** 3
        out.append(row("bmm-bin" if bin_ else "bmm", "bmm_pm1_bin" if bin_ else "bmm_pm1", eng.value.decode(),
                       f"{n}x{n}x{n}", reps, warmup, med.value, mn.value, ops / (med.value * 1e-9), "bitops/s",
                       True))
        n *= 2
    return out


def bconv_rows(bin_, reps, warmup, cmin, cmax, hw=64, batch=16, k=3):
    lib = capi.lib()
    med, mn = C.c_double(), C.c_double()
    eng = C.create_string_buffer(16)
    out = []
    c = cmin
    while c <= cmax:
        capi.check(lib.btnn_cuda_bench_bconv(hw, batch, c, c, k, int(bin_), reps, warmup, C.byref(med), C.byref(mn),
                                             eng, 16))
        ops = 2.0 * hw * hw * batch * c * c * k * k  # border taps counted as full (bench.hpp:290-292)
        out.append(row("bconv-bin" if bin_ else "bconv", "bconv_fused" if bin_ else "bconv_pm1", eng.value.decode(),
                       f"{hw}x{hw}x{batch}x{c}->{c}k{k}", reps, warmup, med.value, mn.value,
                       ops / (med.value * 1e-9), "bitops/s", True))
        c *= 2
    return out


def model_rows(name, batches, reps, warmup, hw=None):
    import torch
    m = M.stock_model(name, hw, hw) if hw else M.stock_model(name)
    ws = W.build_weights(m, W.random_weights(m, 1))
    rng = np.random.default_rng(1)
    # precheck: both bit-GEMM engines give identical logits on one image
    x1 = rng.standard_normal((1, m.in_h, m.in_w, m.in_c), dtype=np.float32)
    capi.set_engine(capi.ENGINE_POPC)
    a, _ = btnn.Plan(m, ws, 1).run(x1)
    capi.set_engine(capi.ENGINE_AUTO)
    b, _ = btnn.Plan(m, ws, 1).run(x1)
    ok = np.array_equal(a.view(np.uint64), b.view(np.uint64))
    lib = capi.lib()
    out = []
    plan = btnn.Plan(m, ws, max(batches))
    for bsz in batches:
        xd = torch.randn((bsz, m.in_h, m.in_w, m.in_c), dtype=torch.float32, device="cuda")
        ld = torch.empty((bsz, m.classes), dtype=torch.float64, device="cuda")
        bd = torch.empty((bsz,), dtype=torch.int32, device="cuda")
        s = torch.cuda.Stream()  # a real stream: plan_run_device treats NULL as "the plan's own stream"

        def step():
            capi.check(lib.btnn_cuda_plan_run_device(plan.h, 0, C.cast(xd.data_ptr(), C.POINTER(C.c_float)), bsz,
                                                     C.cast(ld.data_ptr(), C.POINTER(C.c_double)),
                                                     C.cast(bd.data_ptr(), C.POINTER(C.c_int32)),
                                                     C.c_void_p(s.cuda_stream)))
        for _ in range(warmup):
            step()
        ts = []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            step()
            e1.record(s)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e6)
        med = float(np.median(ts))
        out.append(row("model", m.name, "tc_i8", f"batch{bsz}", reps, warmup, med, float(min(ts)),
                       bsz * 1e9 / med, "img/s", ok))
    return out


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--suite", required=True, choices=["bmm", "bmm-bin", "bconv", "bconv-bin", "model"])
    p.add_argument("--model", default="resnet18")
    p.add_argument("--batches", default="8,16,32,64")
    p.add_argument("--reps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--bmm-max-n", type=int, default=4096)
    p.add_argument("--conv-max-c", type=int, default=2048)
    p.add_argument("--seed", type=int, default=1)
    p.add_argument("--csv", default="-")
    a = p.parse_args()
    if a.suite in ("bmm", "bmm-bin"):
        rows = bmm_rows(a.suite == "bmm-bin", a.reps, a.warmup, 128, a.bmm_max_n)
    elif a.suite in ("bconv", "bconv-bin"):
        rows = bconv_rows(a.suite == "bconv-bin", a.reps, a.warmup, 128, a.conv_max_c)
    else:
        rows = model_rows(a.model, [int(b) for b in a.batches.split(",")], a.reps, a.warmup)
    text = f"# seed={a.seed}\n{HDR}\n" + "\n".join(rows) + "\n"
    if a.csv == "-":
        sys.stdout.write(text)
    else:
        open(a.csv, "w").write(text)


if __name__ == "__main__":
    main()
