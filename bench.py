"""bench.py — BNN inference throughput on 1..N B200s (BASELINE configs 1-5).

Contract:
  python bench.py [--gpus N] [--steps K] [--warmup W] [--model M] [--batch B] [--impl ours|reference]
M = resnet18 (default, batch 512: BASELINE config 5), alexnet (1024), cifar-vgg (1024 or 256),
mnist-mlp (1024), or bmm1024 (config 1: one 1024^3 bmm_pm1 from packed operands).
A step = one forward of the whole network over one synthetic batch of B images per GPU
(weak scaling), through the plan's CUDA graph. `value` times K steps with inputs already
resident in HBM (CUDA events on the launching stream, barrier + synchronize on both
sides, max over ranks); `e2e` times the same K steps through the C-ABI call a user makes
(btnn_cuda_plan_run: pinned host input -> H2D -> network -> D2H logits+labels).
`parity` compares the timed batch's first images with the reference's run_inference
(oracle/_ref) on the same inputs, bit for bit. Rank 0 prints one JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# PAPER.md:708 (RTX 2080, BTC-FMT): context only, not vs_baseline (no published B200 number)
PAPER_IMG_S = {"resnet18": 5.55e3, "alexnet": 3.77e3, "cifar-vgg": 3.85e4, "mnist-mlp": 5.48e6}
DEFAULT_BATCH = {"resnet18": 512, "alexnet": 1024, "cifar-vgg": 1024, "mnist-mlp": 1024, "bmm1024": 1024}
PARITY_IMAGES = {"resnet18": 32, "alexnet": 16, "cifar-vgg": 256, "mnist-mlp": 1024}
SHAPE = {"resnet18": "ImageNet 224x224", "alexnet": "ImageNet 224x224", "cifar-vgg": "CIFAR 32x32",
         "mnist-mlp": "MNIST 28x28"}


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--batch", type=int, default=0, help="images per GPU per step (0: the model's default)")
    p.add_argument("--model", default="resnet18", choices=sorted(DEFAULT_BATCH))
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-kernels", action="store_true", help="skip the kernel-suite sub-benchmarks")
    p.add_argument("--cpu-seconds", type=float, default=12.0)
    return p.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class Clocks:
    """Samples nvidia-smi clocks/throttle reasons during the timed region."""

    def __init__(self, index: int):
        self.index, self.samples, self._stop = index, [], threading.Event()
        self.t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}", "--format=csv,noheader,nounits"],
                                     capture_output=True, text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([s.strip() for s in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self.t.join(timeout=6)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if len(s) > 2 + i and s[2 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None, "reasons": reasons}


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


def engine_peaks():
    """Measured engine peaks on this B200 pool (profiles/microbench_r01.json)."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "microbench_r01.json")))
        return {"b1_mma_sync_tops": d["b1_mma_sync"]["t_bitops"], "tc_i8_tops": d["tc_i8_tmemA_n256"]["tops"],
                "popc_tops": d["popc"]["t_bitops"], "dfma_tflops": d["dfma"]["tflops"]}
    except Exception:
        return {}


def measured_traffic(key):
    """dram__bytes_read.sum + dram__bytes_write.sum per image of the kernel behind layer key,
    from the ncu capture summarized in profiles/traffic.json (None if absent)."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            d = json.load(f)
        return d.get(key)
    except Exception:
        return None


def roofline(m, B, i, ms, engine, plan=None):
    """Roofline of layer i from its measured device time: algorithmic work per launch
     / duration, against the measured peak of the bounding unit."""
    L = m.layers[i]
    hbm = peaks().get("hbm_gbs")
    pk = engine_peaks()
    sec = ms / 1e3
    hbm_line = lambda byts, note: {"bound": "hbm", "kernel": f"layer{i}:{engine}", "achieved": byts / sec / 1e9,
                                   "peak": hbm, "unit": "GB/s", "frac": byts / sec / 1e9 / hbm if hbm else None,
                                   "traffic": None, "peak_source": "MEASURED_PEAKS.json hbm_gbs",
                                   "algorithmic_bytes": byts, "note": note}
    if L.kind == 0 and engine.startswith("tc_i8"):
        # tensor-core first layer (exact integer digits): HBM-bound on its algorithmic bytes —
        # the f32 input read once, the f64 tap and the packed output bits written once.
        byts = B * (4.0 * L.in_h * L.in_w * L.in_channels
                    + (8.0 * L.out_h * L.out_w * L.out_channels if L.residual_out else 0.0)
                    + L.out_h * L.out_w * ((L.out_channels + 127) // 128) * 16.0)
        return hbm_line(byts, "f32 input + f64 tap + bits per image (DESIGN.md §3)")
    if L.kind == 0:  # f64 first layer: 2 flops per tap term
        flops = 2.0 * L.out_h * L.out_w * B * L.in_channels * L.out_channels * L.kh * L.kw
        a = flops / sec / 1e12
        return {"bound": "fp64", "kernel": f"layer{i}:{engine}", "achieved": a, "peak": pk.get("dfma_tflops"),
                "unit": "TFLOP/s", "frac": a / pk["dfma_tflops"] if pk else None, "traffic": None,
                "peak_source": "profiles/microbench_r01.json dfma"}
    if L.kind == 2:  # or_pool: packed bits in and out
        cw = (L.in_channels + 127) // 128 * 16.0
        byts = B * cw * (L.in_h * L.in_w + L.out_h * L.out_w)
        return hbm_line(byts, "packed input + output bits")
    if L.kind == 1 and (L.residual_in or L.residual_out):
        # bn-route conv: the f64 taps dominate: 8 B per output written, 8 B per residual read
        # (the producer's pre-averaged tap when it stored one — the plan reads that, 1x)
        outs = L.out_h * L.out_w * B * L.out_channels
        rd = 0.0
        if L.residual_in:
            src = m.layers[L.shortcut_from]
            halved_by_producer = plan is not None and plan.tap_dims(L.shortcut_from)[2] == 1
            reads = 4 if (src.out_h != L.out_h and not halved_by_producer) else 1
            rd = 8.0 * outs * reads * min(src.out_channels, L.out_channels) / L.out_channels
        wr = 0.0
        if L.residual_out:
            wr = 8.0 * outs / (4 if plan is not None and plan.tap_dims(i)[2] == 1 else 1)
        return hbm_line(wr + rd, "f64 tap written + residual read per launch")
    if L.kind == 1:
        ops = 2.0 * L.out_h * L.out_w * B * L.in_channels * L.out_channels * L.kh * L.kw
    else:
        ops = 2.0 * B * L.in_channels * L.units
    a = ops / sec / 1e12
    peak = pk.get("tc_i8_tops") if engine.startswith("tc_i8") else pk.get("popc_tops")
    return {"bound": "tensor" if engine.startswith("tc_i8") else "int", "kernel": f"layer{i}:{engine}",
            "achieved": a, "peak": peak, "unit": "TFLOP/s", "frac": a / peak if peak else None, "traffic": None,
            "note": "bit-ops (1 MAC = 2 ops) vs the measured tcgen05 kind::i8 peak",
            "peak_source": "profiles/microbench_r01.json"}


def kernel_suites(reps=10, warmup=3):
    """The reference's bmm / bmm-bin / bconv-bin suites (bench.hpp:129-299) at the BASELINE
    points, device-timed through the C ABI: T bit-op/s and fractions of the measured b1
    (emulated mma.sync) peak and of the engine's own (tcgen05 kind::i8) peak. bmm rows time
    the whole call from packed operands (B's tensor-core operand re-expanded each time) and
    the GEMM kernel alone."""
    import ctypes as C

    from paper_2006_16578_b200 import capi

    lib = capi.lib()
    pk = engine_peaks()
    out = {}
    med, mn, kern = C.c_double(), C.c_double(), C.c_double()
    eng = C.create_string_buffer(16)
    for name, bin_ in (("bmm_1024", 0), ("bmm_bin_1024", 1)):
        rb = capi.BenchReadback(None, None, None, C.pointer(kern), None)
        capi.check(lib.btnn_cuda_bench_bmm(1024, bin_, reps, warmup, C.byref(med), C.byref(mn), eng, 16, C.byref(rb)))
        out[name] = {"median_us": med.value / 1e3, "t_bitops": 2 * 1024 ** 3 / med.value / 1e3,
                     "kernel_median_us": kern.value / 1e3, "kernel_t_bitops": 2 * 1024 ** 3 / kern.value / 1e3,
                     "engine": eng.value.decode()}
    # bconv-bin at the paper's Fig. sweep point C=O=512, 64x64, batch 16, K3 (bench.hpp:39-43)
    for c in (128, 512, 2048):
        capi.check(lib.btnn_cuda_bench_bconv(64, 16, c, c, 3, 1, reps, warmup, C.byref(med), C.byref(mn), eng, 16,
                                             None))
        tops = 2 * 64 * 64 * 16 * c * c * 9 / med.value / 1e3
        out[f"bconv_bin_c{c}"] = {"median_us": med.value / 1e3, "t_bitops": tops, "engine": eng.value.decode()}
    for v in out.values():
        if pk:
            v["frac_of_b1_peak"] = v["t_bitops"] / pk["b1_mma_sync_tops"]
            v["frac_of_tc_i8_peak"] = v["t_bitops"] / pk["tc_i8_tops"]
    return out


# ------------------------------------------------------------------ CPU reference arm
def _ref_lib():
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_lib import ref, ref_variant
    r = ref()
    return r, (ref_variant() if r is not None else None)


def ref_run(m, ws, x):
    """The reference's run_inference (oracle/_ref, all host threads) on host images x —
    the checker of the in-run parity field (test infrastructure, never the measured path)."""
    import ctypes as C

    r, _ = _ref_lib()
    if r is None:
        return None
    from oracle_lib import ptr
    spec, store = m.c_spec(), ws.c_store()
    n = x.shape[0]
    lg = np.zeros(n * m.classes)
    lb = np.zeros(n, np.int32)
    st = r.ref_run_store(C.byref(spec), C.byref(store), ptr(np.ascontiguousarray(x), C.c_float), n,
                         ptr(lg, C.c_double), ptr(lb, C.c_int32))
    assert st == 0, r.ref_last_error()
    return lg.reshape(n, m.classes), lb


def cpu_reference(model_name: str, seconds: float, seed: int = 1, steps: int = 3, warmup: int = 0):
    """Times the reference's own run_inference (oracle/_ref, all host threads): `warmup`
    untimed and `steps` timed steps, each a bounded sample of the workload sized so the
    timed steps take about `seconds` in total; returns (img/s, cores, sample description)."""
    import ctypes as C

    from paper_2006_16578_b200 import model as M
    from paper_2006_16578_b200 import weights as W

    r, variant = _ref_lib()
    if r is None:
        return None
    from oracle_lib import ptr
    cores = os.cpu_count() or 1
    os.environ["BTNN_THREADS"] = str(cores)
    if model_name == "bmm1024":  # bmm_pm1 1024^3 on packed words (bench.hpp:129-200), bit-op/s
        rng = np.random.default_rng(seed)
        A = rng.integers(0, 2**64, 1024 * 16, dtype=np.uint64)
        Bw = rng.integers(0, 2**64, 1024 * 16, dtype=np.uint64)
        from paper_2006_16578_b200 import capi
        da, db = capi.MatrixDesc(1024, 1024, capi.ROW_PACKED, 8, 128), capi.MatrixDesc(1024, 1024, capi.COL_PACKED, 8, 128)
        out = np.zeros(1024 * 1024, np.int32)

        def one():
            t0 = time.perf_counter()
            assert r.ref_bmm(1, C.byref(da), ptr(A, C.c_uint64), C.byref(db), ptr(Bw, C.c_uint64), capi.BMM_BLOCKED, 0,
                             None, None, 0, out.ctypes.data_as(C.c_void_p)) == 0
            return time.perf_counter() - t0
        t1 = one()
        reps = max(3, min(200, int(seconds / max(t1, 1e-4) / max(1, steps))))
        for _ in range(warmup):
            one()
        times = [one() for _ in range(reps * max(1, steps))]
        med = float(np.median(times))
        return (2 * 1024 ** 3 / med, cores,
                f"bmm_pm1 1024^3 Blocked, median of {len(times)} calls after {warmup} warm-up, libbtnn_ref_{variant}")
    m = M.stock_model(model_name)
    ws = W.build_weights(m, W.random_weights(m, seed))
    spec, store = m.c_spec(), ws.c_store()
    rng = np.random.default_rng(seed)

    def run(nimg):
        x = rng.standard_normal((nimg, m.in_h, m.in_w, m.in_c), dtype=np.float32)
        lg = np.zeros(nimg * m.classes)
        lb = np.zeros(nimg, np.int32)
        t0 = time.perf_counter()
        st = r.ref_run_store(C.byref(spec), C.byref(store), ptr(x, C.c_float), nimg, ptr(lg, C.c_double),
                             ptr(lb, C.c_int32))
        dt = time.perf_counter() - t0
        assert st == 0, r.ref_last_error()
        return dt

    t1 = run(min(cores, 8))  # rate estimate
    rate = min(cores, 8) / t1
    steps = max(1, steps)
    nimg = max(cores, int(rate * seconds / steps))
    for _ in range(warmup):
        run(nimg)
    times = [run(nimg) for _ in range(steps)]
    return (nimg * steps / float(sum(times)), cores,
            f"{model_name} {SHAPE.get(model_name, '')}, {nimg} images per step, {steps} timed steps after {warmup} "
            f"warm-up, libbtnn_ref_{variant}")


def metric_of(model):
    if model == "bmm1024":
        return "bmm_pm1 1024x1024x1024 bit-op/s (packed +-1 operands, int32 out)", "bit-ops/s"
    return f"{model} images/s ({SHAPE[model]}, BNN inference)", "images/s"


# ------------------------------------------------------------------ GPU arm
def h2d_ceiling(nbytes, dev):
    """Measured pinned host -> device copy rate (GB/s) for a buffer of the step's input size."""
    import torch
    nb = int(min(nbytes, 1 << 30))
    src = torch.empty(nb, dtype=torch.uint8).pin_memory()
    dst = torch.empty(nb, dtype=torch.uint8, device=dev)
    for _ in range(2):
        dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    for _ in range(5):
        dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize(dev)
    return 5 * nb / (time.perf_counter() - t0) / 1e9


def run_bmm(a, rank, world, local, dist):
    """BASELINE config 1: bmm_pm1 1024^3 from packed operands resident in HBM (value), and
    through the C ABI with host buffers (e2e)."""
    import ctypes as C

    import torch

    from paper_2006_16578_b200 import btnn, capi
    from paper_2006_16578_b200 import dist as D

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    lib = capi.lib()
    n = 1024
    med, mn, kern, strm, grph = C.c_double(), C.c_double(), C.c_double(), C.c_double(), C.c_double()
    eng = C.create_string_buffer(16)
    A = np.zeros(n * 16, np.uint64)
    Bw = np.zeros(n * 16, np.uint64)
    res = np.zeros(n * n, np.int32)
    rb = capi.BenchReadback(A.ctypes.data_as(C.POINTER(C.c_uint64)), Bw.ctypes.data_as(C.POINTER(C.c_uint64)),
                            res.ctypes.data_as(C.c_void_p), C.pointer(kern), C.pointer(strm), C.pointer(grph))
    if dist:
        dist.barrier()
    with Clocks(local) as clk:
        capi.check(lib.btnn_cuda_bench_bmm(n, 0, a.steps, a.warmup, C.byref(med), C.byref(mn), eng, 16, C.byref(rb)))
    # value: one job of K calls submitted as one CUDA graph (device time per call); the same K
    # calls launched back to back from the host (stream_us, bounded by the host launch rate)
    # and the per-call median with events around each call are reported beside it
    call_ns = D.max_over_ranks(grph.value, dev) if dist else grph.value
    value = world * 2 * n ** 3 / (call_ns * 1e-9)
    # e2e: the C-ABI bmm_pm1 with host operands (H2D of A and B, D2H of the int32 result)
    da, db = capi.MatrixDesc(n, n, capi.ROW_PACKED, 8, 128), capi.MatrixDesc(n, n, capi.COL_PACKED, 8, 128)
    e2e_warm = max(3, a.warmup)
    t0 = time.perf_counter()
    for _ in range(e2e_warm):
        got = btnn.bmm_pm1(da, A, db, Bw)
    per_call = (time.perf_counter() - t0) / e2e_warm
    e2e_steps = max(a.steps, min(2000, int(0.25 / max(per_call, 1e-6))))  # (>= ~0.25 s of calls)
    if dist:
        e2e_steps = int(D.max_over_ranks(float(e2e_steps), dev))
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        got = btnn.bmm_pm1(da, A, db, Bw)
    e2e_s = (time.perf_counter() - t0) / e2e_steps
    if dist:
        e2e_s = D.max_over_ranks(e2e_s, dev)
    # parity: the timed call's result and the e2e result vs the reference's bmm_pm1
    parity = None
    r, _ = _ref_lib()
    if r is not None:
        from oracle_lib import ptr
        want = np.zeros(n * n, np.int32)
        assert r.ref_bmm(1, C.byref(da), ptr(A, C.c_uint64), C.byref(db), ptr(Bw, C.c_uint64), capi.BMM_BLOCKED, 0,
                         None, None, 0, want.ctypes.data_as(C.c_void_p)) == 0
        parity = {"entries": n * n, "bit_exact": bool(np.array_equal(res, want) and
                                                      np.array_equal(got.reshape(-1), want)),
                  "checker": "oracle/_ref bmm_pm1 (the reference compiled from its headers)"}
    pk = engine_peaks()
    kops = 2 * n ** 3 / (kern.value * 1e-9) / 1e12
    if rank != 0:
        return
    cpu = None
    if not a.no_cpu_baseline and world == 1:
        rr = cpu_reference("bmm1024", a.cpu_seconds / 4)
        if rr:
            cpu = {"value": rr[0], "unit": "bit-ops/s", "cores": rr[1], "kind": "reference", "sample": rr[2]}
    metric, unit = metric_of("bmm1024")
    print(json.dumps({
        "metric": metric, "value": value, "unit": unit, "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
        "ms_per_step": call_ns / 1e6, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "u1/i32", "data": "synthetic", "impl": "ours",
        "config": {"workload": "bmm_pm1 1024^3, random packed words (bench.hpp:76-87), device-resident operands; "
                               "both operands expanded on chip every call (one kernel per call); K calls "
                               "replayed as one CUDA graph", "global_batch": world,
                   "parallelism": f"dp{world} (independent calls)", "l2": "operands fit L2 (config as stated)"},
        "e2e": {"value": world * 2 * n ** 3 / e2e_s, "unit": unit, "h2d_bytes_per_step": int(A.nbytes + Bw.nbytes),
                "d2h_bytes_per_step": int(res.nbytes), "steps": e2e_steps, "warmup": e2e_warm},
        "gpu_launches": a.steps,
        "roofline": {"bound": "tensor", "kernel": f"bmm_tc_kernel ({eng.value.decode()}, one kernel per call) 1024^3", "achieved": kops,
                     "peak": pk.get("tc_i8_tops"), "unit": "TFLOP/s",
                     "frac": kops / pk["tc_i8_tops"] if pk else None, "traffic": None,
                     "kernel_us": kern.value / 1e3, "call_us": call_ns / 1e3, "stream_us": strm.value / 1e3,
                     "call_median_us": med.value / 1e3,
                     "note": "bit-ops (1 MAC = 2 ops) of the GEMM kernel alone vs the measured tcgen05 kind::i8 peak"},
        "parity": parity, "clocks": clk.summary(), "cpu_baseline": cpu}))


def run_model(a, rank, world, local, dist):
    import ctypes as C

    import torch

    from paper_2006_16578_b200 import btnn, capi
    from paper_2006_16578_b200 import dist as D
    from paper_2006_16578_b200 import model as M
    from paper_2006_16578_b200 import weights as W

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    m = M.stock_model(a.model)
    ws = W.build_weights(m, W.random_weights(m, 1))
    B = a.batch
    plan = btnn.Plan(m, ws, B, devices=(local,))
    bits, f64 = m.bit_macs_per_image()
    gen = torch.Generator(device=dev).manual_seed(1000 + rank)
    x = torch.randn((B, m.in_h, m.in_w, m.in_c), device=dev, dtype=torch.float32, generator=gen)
    logits = torch.empty((B, m.classes), device=dev, dtype=torch.float64)
    labels = torch.empty((B,), device=dev, dtype=torch.int32)
    stream = torch.cuda.Stream(dev)  # non-default: its handle orders the plan's graph
    torch.cuda.set_stream(stream)
    in_bytes = B * m.in_h * m.in_w * m.in_c * 4
    # between timed steps: inputs larger than L2 for the ImageNet models; the small-input
    # models flush L2 with a 256 MB write after every step (the flush is outside the timing)
    flush = None if in_bytes > (200 << 20) else torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def step():
        plan.run_device(x.data_ptr(), B, logits.data_ptr(), labels.data_ptr(), stream.cuda_stream)

    for _ in range(a.warmup):
        step()
    torch.cuda.synchronize(dev)
    if dist:
        dist.barrier()
    torch.cuda.synchronize(dev)
    torch.cuda.profiler.start()  # (ncu --profile-from-start off captures the timed steps only)
    with Clocks(local) as clk:
        if flush is None:
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ev0.record(stream)
            for _ in range(a.steps):
                step()
            ev1.record(stream)
            torch.cuda.synchronize(dev)
            ms = ev0.elapsed_time(ev1)
        else:
            ms = 0.0
            for _ in range(a.steps):
                flush.fill_(1)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                step()
                e1.record(stream)
                torch.cuda.synchronize(dev)
                ms += e0.elapsed_time(e1)
    torch.cuda.profiler.stop()
    if dist:
        dist.barrier()
        ms = D.max_over_ranks(ms, dev)
    ms_per_step = ms / a.steps
    value = B * world * a.steps / (ms / 1e3)
    launches = plan.launches(B)

    # ---- in-run parity: the timed batch's first images vs the reference's run_inference
    parity = None
    k = min(B, PARITY_IMAGES.get(a.model, 16))
    if rank == 0:
        xh0 = x[:k].cpu().numpy()
        want = ref_run(m, ws, xh0)
        if want is not None:
            got_l, got_b = logits[:k].cpu().numpy(), labels[:k].cpu().numpy()
            parity = {"images": k, "of_batch": B,
                      "bit_exact": bool(np.array_equal(got_l.view(np.uint64), want[0].view(np.uint64))
                                        and np.array_equal(got_b, want[1])),
                      "checker": "oracle/_ref run_inference (the reference compiled from its headers)"}

    # ---- e2e through the C-ABI call with pinned host buffers
    xh = torch.randn((B, m.in_h, m.in_w, m.in_c), dtype=torch.float32).pin_memory()
    lh = torch.empty((B, m.classes), dtype=torch.float64).pin_memory()
    bh = torch.empty((B,), dtype=torch.int32).pin_memory()
    lib = capi.lib()

    def e2e_step():
        capi.check(lib.btnn_cuda_plan_run(plan.h, C.cast(xh.data_ptr(), C.POINTER(C.c_float)), B,
                                          C.cast(lh.data_ptr(), C.POINTER(C.c_double)),
                                          C.cast(bh.data_ptr(), C.POINTER(C.c_int32))))

    # host-timed: at least W warm-up calls (the first captures the chunk graphs and calibrates
    # the input pipeline) and at least K timed calls, more when K calls take under ~0.25 s (the
    # small-input models' ~0.1-1.5 ms calls: a 20-call window is host-noise dominated)
    e2e_warm = max(3, a.warmup)
    t0 = time.perf_counter()
    for _ in range(e2e_warm):
        e2e_step()
    per_call = (time.perf_counter() - t0) / e2e_warm
    e2e_steps = max(a.steps, min(2000, int(0.25 / max(per_call, 1e-6))))
    if dist:  # (every rank times the same number of calls)
        e2e_steps = int(D.max_over_ranks(float(e2e_steps), dev))
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        e2e_step()
    e2e_s = time.perf_counter() - t0
    if dist:
        e2e_s = D.max_over_ranks(e2e_s, dev)
    e2e = B * world * e2e_steps / e2e_s
    h2d = h2d_ceiling(in_bytes, dev)

    # ---- per-layer device times (separate timed pass, per-layer CUDA events)
    plan.set_breakdown(True)
    nb = max(3, a.steps // 4)
    layer_ms = np.zeros(len(m.layers))
    for _ in range(nb):
        plan.run(xh.numpy())
        layer_ms += plan.layer_ms()
    plan.set_breakdown(False)
    layer_ms /= nb
    engines = plan.engines()
    top = int(np.argmax(layer_ms))
    roof = roofline(m, B, top, layer_ms[top], engines[top], plan)
    roof["share_of_step"] = float(layer_ms[top] / layer_ms.sum())
    # every layer against its own bound; the network's composite roofline fraction is the time
    # the layers would take at their bounds over the time they take (layers without a bound:
    # their measured time counts on both sides)
    per_layer, ideal = [], 0.0
    for i, L in enumerate(m.layers):
        # (an or_pool fused into its producer's epilogue does no work of its own)
        r = roofline(m, B, i, layer_ms[i], engines[i], plan) if layer_ms[i] > 0 and engines[i] != "fused" else {}
        f = r.get("frac")
        per_layer.append({"layer": i, "engine": engines[i], "ms": float(layer_ms[i]), "bound": r.get("bound"),
                          "achieved": r.get("achieved"), "unit": r.get("unit"), "frac": f})
        ideal += layer_ms[i] * (f if f else 1.0)
    network_roofline = {"frac": float(ideal / layer_ms.sum()), "ideal_ms": float(ideal),
                        "measured_ms": float(layer_ms.sum()), "layers": per_layer}
    tr = measured_traffic(f"{a.model}:layer{top}:{engines[top]}") or (
        measured_traffic(f"layer{top}:{engines[top]}") if a.model == "resnet18" else None)
    if tr is not None:  # DRAM bytes per launch from the committed ncu capture, scaled to B
        roof["traffic"] = tr["bytes_per_image"] * B
        roof["traffic_source"] = tr["source"]

    if rank == 0:
        cpu = None
        if not a.no_cpu_baseline and world == 1:
            r = cpu_reference(a.model, a.cpu_seconds)
            if r:
                cpu = {"value": r[0], "unit": "images/s", "cores": r[1], "kind": "reference", "sample": r[2]}
        metric, unit = metric_of(a.model)
        out = {"metric": metric, "value": value, "unit": unit,
               "n_gpus": world, "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms_per_step,
               "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u1/i32/f64",
               "data": "synthetic", "impl": "ours",
               "config": {"workload": f"{a.model} {SHAPE[a.model]} forward (BNN inference, random-init weights)",
                          "batch_per_gpu": B, "global_batch": B * world, "parallelism": f"dp{world} (batch shards)",
                          "l2": (f"inputs larger than L2 ({in_bytes / 1e6:.0f} MB/step per GPU)" if flush is None
                                 else "L2 flushed (256 MB write) before every timed step"),
                          "bit_macs_per_image": bits, "f64_macs_per_image": f64},
               "e2e": {"value": e2e, "unit": unit, "h2d_bytes_per_step": int(xh.numel() * 4),
                       "d2h_bytes_per_step": int(lh.numel() * 8 + bh.numel() * 4),
                       "h2d_ceiling_gbs": h2d, "h2d_ceiling_img_s": h2d * 1e9 / (in_bytes / B),
                       "frac_of_h2d_ceiling": e2e / (h2d * 1e9 / (in_bytes / B)),
                       "pipeline": plan.e2e_schedule(B), "steps": e2e_steps, "warmup": e2e_warm},
               "gpu_launches": launches * a.steps,
               "roofline": roof,
               "network_roofline": network_roofline,
               "parity": parity,
               "layer_ms": {f"{i}:{engines[i]}": round(float(t), 4) for i, t in enumerate(layer_ms)},
               "paper_turing_img_s": PAPER_IMG_S.get(a.model),
               "clocks": clk.summary(),
               "cpu_baseline": cpu}
        if a.model == "resnet18" and not a.no_kernels:
            try:
                out["kernels"] = kernel_suites()
            except Exception as ex:  # the model line stays valid even if a suite fails
                out["kernels"] = {"error": str(ex)}
        print(json.dumps(out))
    plan.close()


def main():
    a = parse()
    rank, world, local = dist_env()
    if world != a.gpus and "RANK" in os.environ:
        a.gpus = world
    if not a.batch:
        a.batch = DEFAULT_BATCH[a.model]
    dist = None
    if world > 1:
        import torch.distributed as dist  # noqa: F811
        import torch
        torch.cuda.set_device(local) if a.impl == "ours" else None
        dist.init_process_group("nccl" if a.impl == "ours" else "gloo")

    if a.impl == "reference":
        if rank == 0:
            # the whole --steps K --warmup W run stays within a few minutes: ~1.5x cpu_seconds
            res = cpu_reference(a.model, a.cpu_seconds, steps=a.steps, warmup=a.warmup)
            if res is None:
                print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}))
            else:
                v, cores, sample = res
                metric, unit = metric_of(a.model)
                print(json.dumps({"metric": metric, "value": v, "unit": unit, "n_gpus": a.gpus, "steps": a.steps,
                                  "warmup": a.warmup, "ms_per_step": None, "higher_is_better": True,
                                  "scaling": "weak", "vs_baseline": None, "dtype": "u1/f64", "data": "synthetic",
                                  "impl": "reference",
                                  "config": {"workload": f"{a.model} forward (BNN, reference CPU run_inference)"
                                             if a.model != "bmm1024" else "bmm_pm1 1024^3 (reference CPU)",
                                             "global_batch": None},
                                  "cpu_baseline": {"value": v, "unit": unit, "cores": cores, "kind": "reference",
                                                   "sample": sample},
                                  "e2e": {"value": v, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}))
    elif a.model == "bmm1024":
        run_bmm(a, rank, world, local, dist)
    else:
        run_model(a, rank, world, local, dist)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
