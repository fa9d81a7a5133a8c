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

Every bmm / bconv size also gets an `fsb` row (bench.hpp:140-156, 230-245): the call's
operands are the 8 x 128-tile (FSB / tiled) layouts, converted on the device inside each timed
call (btnn_cuda_bench_bmm_fsb / btnn_cuda_bench_bconv_fsb).

`precheck` follows bench.hpp:164-176 / 248-256: after timing, the device operands and the
result of the timed call are read back and 256 sampled entries are recomputed on the host
from the packed words (the +-1 dot n - 2*popc(a ^ b), bit_buffer.hpp:94-113; for BConv the
in-frame taps and the C*taps - 2*popc rule, bconv.hpp:107-130); the model suite compares the
timed batch's logits (first 32 images) with the reference's run_inference (oracle/_ref).
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


def row(suite, kernel, variant, shape, reps, warmup, med, mn, thr, unit, ok, layout="plain"):
    return (f"{suite},{kernel},{variant},{layout},{shape},0,{reps},{warmup},{med:.1f},{med:.1f},{mn:.1f},"
            f"{thr:.3f},{unit},{'ok' if ok else 'FAIL'}")


SAMPLES = 256


def _popc(x):
    return np.bitwise_count(x).sum(axis=-1).astype(np.int64)


def bmm_precheck(n, bin_, a, b, out, rng):
    """Sampled entries of the timed call's result vs the packed-word dot (bench.hpp:164-176)."""
    kw = a.size // n
    A, Bm = a.reshape(n, kw), b.reshape(n, kw)  # RowPacked rows of A, ColPacked columns of B
    i, j = rng.integers(0, n, SAMPLES), rng.integers(0, n, SAMPLES)
    v = n - 2 * _popc(A[i] ^ Bm[j])
    if not bin_:
        return bool(np.array_equal(out.reshape(n, n)[i, j].astype(np.int64), v))
    bits = (out.reshape(n, kw)[i, j // 64] >> (j % 64).astype(np.uint64)) & np.uint64(1)
    return bool(np.array_equal(bits.astype(bool), v >= 0))


def bmm_rows(bin_, reps, warmup, nmin, nmax):
    lib = capi.lib()
    med, mn = C.c_double(), C.c_double()
    eng = C.create_string_buffer(16)
    out = []
    rng = np.random.default_rng(11)
    n = nmin
    while n <= nmax:
        kw = -(-n // 128) * 2
        a, b = np.zeros(n * kw, np.uint64), np.zeros(n * kw, np.uint64)
        res = np.zeros(n * kw, np.uint64) if bin_ else np.zeros(n * n, np.int32)
        rb = capi.BenchReadback(a.ctypes.data_as(C.POINTER(C.c_uint64)), b.ctypes.data_as(C.POINTER(C.c_uint64)),
                                res.ctypes.data_as(C.c_void_p), None)
        for layout, fn in (("plain", lib.btnn_cuda_bench_bmm), ("fsb", lib.btnn_cuda_bench_bmm_fsb)):
            capi.check(fn(n, int(bin_), reps, warmup, C.byref(med), C.byref(mn), eng, 16, C.byref(rb)))
            ops = 2.0 * n ** 3
            out.append(row("bmm-bin" if bin_ else "bmm", "bmm_pm1_bin" if bin_ else "bmm_pm1", eng.value.decode(),
                           f"{n}x{n}x{n}", reps, warmup, med.value, mn.value, ops / (med.value * 1e-9), "bitops/s",
                           bmm_precheck(n, bin_, a, b, res, rng), layout))
        n *= 2
    return out


def bconv_precheck(hw, batch, c, o, k, bin_, act, filt, res, rng):
    """Sampled outputs (p, q, n, o) of the timed call vs the packed-word BConv rule: over the
    in-frame taps, v = C*taps - 2*popc(x ^ w) (bconv.hpp:107-130; pad bits 0 in both)."""
    npad, cw, opad = -(-batch // 8) * 8, -(-c // 128) * 2, -(-o // 128) * 128
    X = act.reshape(hw, hw, npad, cw)
    Wf = filt.reshape(k, k, -1, cw)
    pad = k // 2
    ok = True
    for _ in range(SAMPLES):
        p, q, n, oo = (int(v) for v in (rng.integers(0, hw), rng.integers(0, hw), rng.integers(0, batch),
                                        rng.integers(0, o)))
        acc, taps = 0, 0
        for r in range(k):
            for s_ in range(k):
                h, w = p + r - pad, q + s_ - pad
                if 0 <= h < hw and 0 <= w < hw:
                    taps += 1
                    acc += int(np.bitwise_count(X[h, w, n] ^ Wf[r, s_, oo]).sum())
        v = c * taps - 2 * acc
        if bin_:
            cwo = opad // 64
            word = int(res.reshape(hw, hw, npad, cwo)[p, q, n, oo // 64])
            ok &= bool((word >> (oo % 64)) & 1) == (v >= 0)
        else:
            ok &= int(res.reshape(hw, hw, batch, o)[p, q, n, oo]) == v
    return bool(ok)


def bconv_rows(bin_, reps, warmup, cmin, cmax, hw=64, batch=16, k=3):
    lib = capi.lib()
    med, mn = C.c_double(), C.c_double()
    eng = C.create_string_buffer(16)
    out = []
    rng = np.random.default_rng(12)
    c = cmin
    while c <= cmax:
        npad, cw = -(-batch // 8) * 8, -(-c // 128) * 2
        act = np.zeros(hw * hw * npad * cw, np.uint64)
        filt = np.zeros(k * k * (-(-c // 8) * 8) * cw, np.uint64)
        res = np.zeros(hw * hw * npad * cw, np.uint64) if bin_ else np.zeros(hw * hw * batch * c, np.int32)
        rb = capi.BenchReadback(act.ctypes.data_as(C.POINTER(C.c_uint64)), filt.ctypes.data_as(C.POINTER(C.c_uint64)),
                                res.ctypes.data_as(C.c_void_p), None)
        for layout, fn in (("plain", lib.btnn_cuda_bench_bconv), ("fsb", lib.btnn_cuda_bench_bconv_fsb)):
            capi.check(fn(hw, batch, c, c, k, int(bin_), reps, warmup, C.byref(med), C.byref(mn), eng, 16, C.byref(rb)))
            ops = 2.0 * hw * hw * batch * c * c * k * k  # border taps counted as full (bench.hpp:290-292)
            out.append(row("bconv-bin" if bin_ else "bconv", "bconv_fused" if bin_ else "bconv_pm1",
                           eng.value.decode(), f"{hw}x{hw}x{batch}x{c}->{c}k{k}", reps, warmup, med.value, mn.value,
                           ops / (med.value * 1e-9), "bitops/s",
                           bconv_precheck(hw, batch, c, c, k, bin_, act, filt, res, rng), layout))
        c *= 2
    return out


def model_precheck(m, ws, xd, ld, bd, k):
    """The timed batch's first k logits / labels vs the reference's run_inference
    (oracle/_ref, test infrastructure used here only as the checker)."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_lib import ptr, ref
    r = ref()
    if r is None:
        return False
    x = xd[:k].cpu().numpy()
    lg = np.zeros(k * m.classes)
    lb = np.zeros(k, np.int32)
    spec, store = m.c_spec(), ws.c_store()
    assert r.ref_run_store(C.byref(spec), C.byref(store), ptr(np.ascontiguousarray(x), C.c_float), k,
                           ptr(lg, C.c_double), ptr(lb, C.c_int32)) == 0
    got = ld[:k].cpu().numpy().reshape(-1)
    return bool(np.array_equal(got.view(np.uint64), lg.view(np.uint64)) and np.array_equal(bd[:k].cpu().numpy(), lb))


def model_rows(name, batches, reps, warmup, hw=None):
    import torch
    m = M.stock_model(name, hw, hw) if hw else M.stock_model(name)
    ws = W.build_weights(m, W.random_weights(m, 1))
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
                       bsz * 1e9 / med, "img/s", model_precheck(m, ws, xd, ld, bd, min(bsz, 32))))
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
