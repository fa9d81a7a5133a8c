"""bench.py — BNN ResNet-18 (ImageNet shape) inference throughput on 1..N B200s.

Contract:
  python bench.py [--gpus N] [--steps K] [--warmup W] [--batch B] [--impl ours|reference]
A step = one forward of the whole network over one synthetic batch of B images per GPU
(weak scaling), through the plan's CUDA graph. `value` times K steps with inputs already
resident in HBM (CUDA events on the launching stream, barrier + synchronize on both
sides, max over ranks); `e2e` times the same K steps through the C-ABI call a user makes
(btnn_cuda_plan_run: pinned host input -> H2D -> network -> D2H logits+labels).
Rank 0 prints one JSON line.
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

PAPER_IMG_S = 5.55e3  # PAPER.md:708 (RTX 2080, batch 512) — context only, not vs_baseline


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--batch", type=int, default=512, help="images per GPU per step")
    p.add_argument("--model", default="resnet18")
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--no-cpu-baseline", action="store_true")
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


def roofline(m, B, i, ms, engine):
    """Roofline of layer i from its measured device time: algorithmic work per launch
     / duration, against the measured peak of the bounding unit."""
    L = m.layers[i]
    hbm = peaks().get("hbm_gbs")
    pk = engine_peaks()
    sec = ms / 1e3
    if L.kind == 0 and engine.startswith("tc_i8"):
        # tensor-core first layer (exact integer digits): HBM-bound on its algorithmic bytes —
        # the f32 input read once, the f64 tap and the packed output bits written once.
        byts = B * (4.0 * L.in_h * L.in_w * L.in_channels
                    + (8.0 * L.out_h * L.out_w * L.out_channels if L.residual_out else 0.0)
                    + L.out_h * L.out_w * ((L.out_channels + 127) // 128) * 16.0)
        a = byts / sec / 1e9
        return {"bound": "hbm", "kernel": f"layer{i}:{engine}", "achieved": a, "peak": hbm, "unit": "GB/s",
                "frac": a / hbm if hbm else None, "traffic": None, "peak_source": "MEASURED_PEAKS.json hbm_gbs",
                "note": "f32 input + f64 tap + bits per image (DESIGN.md §3)"}
    if L.kind == 0:  # f64 first layer: 2 flops per tap term
        flops = 2.0 * L.out_h * L.out_w * B * L.in_channels * L.out_channels * L.kh * L.kw
        a = flops / sec / 1e12
        return {"bound": "fp64", "kernel": f"layer{i}:{engine}", "achieved": a, "peak": pk.get("dfma_tflops"),
                "unit": "TFLOP/s", "frac": a / pk["dfma_tflops"] if pk else None, "traffic": None,
                "peak_source": "profiles/microbench_r01.json dfma"}
    if L.kind == 1 and (L.residual_in or L.residual_out):
        # bn-route conv: the f64 taps dominate: 8 B per output written (+8 or 4x8 read)
        outs = L.out_h * L.out_w * B * L.out_channels
        rd = 0.0
        if L.residual_in:
            src = m.layers[L.shortcut_from]
            rd = 8.0 * outs * (4 if src.out_h != L.out_h else 1) * min(src.out_channels, L.out_channels) / L.out_channels
        byts = 8.0 * outs * (1 if L.residual_out else 0) + rd
        a = byts / sec / 1e9
        return {"bound": "hbm", "kernel": f"layer{i}:{engine}", "achieved": a, "peak": hbm, "unit": "GB/s",
                "frac": a / hbm if hbm else None, "traffic": None, "peak_source": "MEASURED_PEAKS.json hbm_gbs"}
    if L.kind == 1:
        ops = 2.0 * L.out_h * L.out_w * B * L.in_channels * L.out_channels * L.kh * L.kw
    else:
        ops = 2.0 * B * L.in_channels * L.units
    a = ops / sec / 1e12
    peak = pk.get("tc_i8_tops") if engine == "tc_i8" else pk.get("popc_tops")
    return {"bound": "tensor" if engine == "tc_i8" else "int", "kernel": f"layer{i}:{engine}", "achieved": a,
            "peak": peak, "unit": "TFLOP/s", "frac": a / peak if peak else None, "traffic": None,
            "note": "bit-ops (1 MAC = 2 ops)", "peak_source": "profiles/microbench_r01.json"}


def kernel_suites(reps=10, warmup=3):
    """The reference's bmm / bmm-bin / bconv-bin suites (bench.hpp:129-299) at the BASELINE
    points, device-timed through the C ABI: T bit-op/s and fractions of the measured b1
    (emulated mma.sync) peak and of the engine's own (tcgen05 kind::i8) peak."""
    import ctypes as C

    from paper_2006_16578_b200 import capi

    lib = capi.lib()
    pk = engine_peaks()
    out = {}
    med, mn = C.c_double(), C.c_double()
    eng = C.create_string_buffer(16)
    for name, bin_ in (("bmm_1024", 0), ("bmm_bin_1024", 1)):
        capi.check(lib.btnn_cuda_bench_bmm(1024, bin_, reps, warmup, C.byref(med), C.byref(mn), eng, 16))
        tops = 2 * 1024 ** 3 / med.value / 1e3
        out[name] = {"median_us": med.value / 1e3, "t_bitops": tops, "engine": eng.value.decode()}
    # bconv-bin at the paper's Fig. sweep point C=O=512, 64x64, batch 16, K3 (bench.hpp:39-43)
    for c in (128, 512, 2048):
        capi.check(lib.btnn_cuda_bench_bconv(64, 16, c, c, 3, 1, reps, warmup, C.byref(med), C.byref(mn), eng, 16))
        tops = 2 * 64 * 64 * 16 * c * c * 9 / med.value / 1e3
        out[f"bconv_bin_c{c}"] = {"median_us": med.value / 1e3, "t_bitops": tops, "engine": eng.value.decode()}
    for v in out.values():
        if pk:
            v["frac_of_b1_peak"] = v["t_bitops"] / pk["b1_mma_sync_tops"]
            v["frac_of_tc_i8_peak"] = v["t_bitops"] / pk["tc_i8_tops"]
    return out


# ------------------------------------------------------------------ CPU reference arm
def cpu_reference(model_name: str, seconds: float, seed: int = 1, steps: int = 3, warmup: int = 0):
    """Times the reference's own run_inference (oracle/_ref, all host threads): `warmup`
    untimed and `steps` timed steps, each a bounded sample of the workload sized so the
    timed steps take about `seconds` in total; returns (img/s, cores, sample description)."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import ctypes as C

    from oracle_lib import ptr, ref, ref_variant
    from paper_2006_16578_b200 import model as M
    from paper_2006_16578_b200 import weights as W

    r = ref()
    if r is None:
        return None
    cores = os.cpu_count() or 1
    m = M.stock_model(model_name)
    ws = W.build_weights(m, W.random_weights(m, seed))
    spec, store = m.c_spec(), ws.c_store()
    rng = np.random.default_rng(seed)
    os.environ["BTNN_THREADS"] = str(cores)

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
            f"{model_name} 224x224, {nimg} images per step, {steps} timed steps after {warmup} warm-up, "
            f"libbtnn_ref_{ref_variant()}")


# ------------------------------------------------------------------ GPU arm
def main():
    a = parse()
    rank, world, local = dist_env()
    if world != a.gpus and "RANK" in os.environ:
        a.gpus = world
    dist = None
    if world > 1:
        import torch.distributed as dist  # noqa: F811
        import torch
        torch.cuda.set_device(local) if a.impl == "ours" else None
        dist.init_process_group("nccl" if a.impl == "ours" else "gloo")

    if a.impl == "reference":
        if rank != 0:
            return
        # the whole --steps K --warmup W run stays within a few minutes: ~1.5x cpu_seconds
        res = cpu_reference(a.model, a.cpu_seconds, steps=a.steps, warmup=a.warmup)
        if res is None:
            print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}))
            return
        v, cores, sample = res
        print(json.dumps({"metric": f"{a.model} images/s (ImageNet 224x224, BNN inference)", "value": v,
                          "unit": "images/s", "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup,
                          "ms_per_step": None,
                          "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u1/f64",
                          "data": "synthetic", "impl": "reference",
                          "config": {"workload": f"{a.model} 224x224x3 forward (BNN, reference CPU run_inference)",
                                     "global_batch": None},
                          "cpu_baseline": {"value": v, "unit": "images/s", "cores": cores, "kind": "reference",
                                           "sample": sample},
                          "e2e": {"value": v, "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}))
        return

    import torch

    from paper_2006_16578_b200 import btnn
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

    def step():
        plan.run_device(x.data_ptr(), B, logits.data_ptr(), labels.data_ptr(), stream.cuda_stream)

    for _ in range(a.warmup):
        step()
    torch.cuda.synchronize(dev)
    if dist:
        dist.barrier()
    torch.cuda.synchronize(dev)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        ev0.record(stream)
        for _ in range(a.steps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize(dev)
    if dist:
        dist.barrier()
    ms = ev0.elapsed_time(ev1)
    if dist:
        ms = D.max_over_ranks(ms, dev)
    ms_per_step = ms / a.steps
    value = B * world * a.steps / (ms / 1e3)
    launches = plan.launches(B)

    # ---- e2e through the C-ABI call with pinned host buffers
    xh = torch.randn((B, m.in_h, m.in_w, m.in_c), dtype=torch.float32).pin_memory()
    lh = torch.empty((B, m.classes), dtype=torch.float64).pin_memory()
    bh = torch.empty((B,), dtype=torch.int32).pin_memory()
    import ctypes as C

    from paper_2006_16578_b200 import capi

    lib = capi.lib()

    def e2e_step():
        capi.check(lib.btnn_cuda_plan_run(plan.h, C.cast(xh.data_ptr(), C.POINTER(C.c_float)), B,
                                          C.cast(lh.data_ptr(), C.POINTER(C.c_double)),
                                          C.cast(bh.data_ptr(), C.POINTER(C.c_int32))))

    for _ in range(max(1, a.warmup // 2)):
        e2e_step()
    if dist:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(a.steps):
        e2e_step()
    e2e_s = time.perf_counter() - t0
    if dist:
        e2e_s = D.max_over_ranks(e2e_s, dev)
    e2e = B * world * a.steps / e2e_s

    # ---- per-layer device times (separate timed pass, per-layer CUDA events)
    plan.set_breakdown(True)
    layer_ms = np.zeros(len(m.layers))
    for _ in range(max(3, a.steps // 4)):
        plan.run(xh.numpy())
        layer_ms += plan.layer_ms()
    plan.set_breakdown(False)
    layer_ms /= max(3, a.steps // 4)
    engines = plan.engines()
    top = int(np.argmax(layer_ms))
    roof = roofline(m, B, top, layer_ms[top], engines[top])
    roof["share_of_step"] = float(layer_ms[top] / layer_ms.sum())
    tr = measured_traffic(f"layer{top}:{engines[top]}")
    if tr is not None:  # DRAM bytes per launch from the committed ncu capture, scaled to B
        roof["traffic"] = tr["bytes_per_image"] * B
        roof["traffic_source"] = tr["source"]

    out = None
    if rank == 0:
        cpu = None
        if not a.no_cpu_baseline and world == 1:
            r = cpu_reference(a.model, a.cpu_seconds)
            if r:
                cpu = {"value": r[0], "unit": "images/s", "cores": r[1], "kind": "reference", "sample": r[2]}
        out = {"metric": f"{a.model} images/s (ImageNet 224x224, BNN inference)", "value": value, "unit": "images/s",
               "n_gpus": world, "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms_per_step,
               "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u1/i32/f64",
               "data": "synthetic", "impl": "ours",
               "config": {"workload": f"{a.model} 224x224x3 forward (BNN, bit-exact vs reference)",
                          "batch_per_gpu": B, "global_batch": B * world, "parallelism": f"dp{world} (batch shards)",
                          "l2": f"inputs larger than L2 ({B * m.in_h * m.in_w * m.in_c * 4 / 1e6:.0f} MB/step per GPU)",
                          "bit_macs_per_image": bits, "f64_macs_per_image": f64},
               "e2e": {"value": e2e, "unit": "images/s", "h2d_bytes_per_step": int(xh.numel() * 4),
                       "d2h_bytes_per_step": int(lh.numel() * 8 + bh.numel() * 4)},
               "gpu_launches": launches * a.steps,
               "roofline": roof,
               "layer_ms": {f"{i}:{engines[i]}": round(float(t), 4) for i, t in enumerate(layer_ms)},
               "paper_turing_img_s": PAPER_IMG_S,
               "clocks": clk.summary(),
               "cpu_baseline": cpu}
        try:
            out["kernels"] = kernel_suites()
        except Exception as ex:  # the model line stays valid even if a suite fails
            out["kernels"] = {"error": str(ex)}
        print(json.dumps(out))
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    plan.close()


if __name__ == "__main__":
    main()
