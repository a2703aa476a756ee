#!/usr/bin/env python
"""bench.py — 2-bit LUT-GEMM/conv TOPS (2*M*N*K/s) and % of roofline on B200.

Default workload (BASELINE.json configs[2]): every 1x1 and 3x3 conv of ResNet-50 (52
LUT convs, 224x224 input) at batch 256 PER GPU (weak scaling: ranks take disjoint
image shards; no data-path collective).  One step = all 52 layers, each im2col (S3)
-> LUT GEMM + fused requant (S5-S7) over per-layer independent inputs already resident
in HBM (reading Q16).  Other workloads: --workload vgg16 | gemm (config 5, square GEMM
with an output-channel split and an NCCL all-gather of the int32 C).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

Prints ONE JSON line on rank 0.  Timing: CUDA-graph replay of the step, CUDA events on
the launching stream, barrier + synchronize on both sides, max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

MEASURED = os.path.join(ROOT, "MEASURED_PEAKS.json")
TRAFFIC = os.path.join(ROOT, "profiles", "traffic.json")
METRIC = "2-bit LUT-GEMM/conv TOPS (2MNK/s) and % of roofline"


# ---------------------------------------------------------------- helpers
def peaks():
    """Roofline denominators: measured HBM copy bandwidth and the int8 dense tensor peak
    derived from the measured bf16 cuBLAS peak x the nominal int8/bf16 ratio (4.5/2.25 = 2)."""
    d = {}
    if os.path.exists(MEASURED):
        with open(MEASURED) as f:
            d = json.load(f)
        src = "measured (MEASURED_PEAKS.json)"
    else:
        d = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}
        src = "fallback (B200_PROFILING.md)"
    return {"hbm_gbs": d["hbm_gbs"], "i8_burst": 2 * d["bf16_tflops"],
            "i8_sustained": 2 * d.get("bf16_tflops_sustained", d["bf16_tflops"]), "src": src}


class ClockSampler:
    """Samples SM clock and clock-event reasons via NVML during the timed region."""

    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:  # pragma: no cover - no NVML
            self.nv = None
        self.names = {}
        if self.nv:
            nv = self.nv
            self.names = {nv.nvmlClocksEventReasonHwSlowdown: "hw_slowdown",
                          nv.nvmlClocksEventReasonHwThermalSlowdown: "hw_thermal_slowdown",
                          nv.nvmlClocksEventReasonSwThermalSlowdown: "sw_thermal_slowdown",
                          nv.nvmlClocksEventReasonSwPowerCap: "sw_power_cap",
                          nv.nvmlClocksEventReasonHwPowerBrakeSlowdown: "hw_power_brake_slowdown",
                          nv.nvmlClocksEventReasonApplicationsClocksSetting: "applications_clocks_setting"}

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.names.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": len(self.samples)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def max_over_ranks(v: float, ws: int) -> float:
    from paper_2304_09049_b200 import shard
    return shard.max_over_ranks(v, ws, device="cuda")


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


def cpu_info():
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    try:
        cores = len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        cores = os.cpu_count() or 1
    return model, cores


def i8_mma_ceiling(sm_mhz):
    """The kind::i8 instruction's own rate: one 128x128x32 MMA per 64 SM cycles (tools/mma_bench.cu,
    profiles/r01_mma_issue_bench.txt: 4418 TOPS measured chip-wide) = 16384 ops/clk/SM, at the SM
    clock observed during the timed region."""
    return 16384 * 148 * (sm_mhz or 1965.0) * 1e6 / 1e12


# ---------------------------------------------------------------- oracle (CPU) legs
def oracle_conv_sample(cfg, runner_layers, image, budget_s=25.0, check=None):
    """Run the plain CPU oracle on one image through the given layers (cpu_baseline leg;
    oracle/ is test infrastructure and is only called here, never on the product path).
    If `check` (layer index -> GPU codes for this image) is given, compare bit-exactly.
    Returns (ops, seconds, layers_done, mismatches)."""
    import oracle
    import synth
    T = oracle.build_lut16(synth.WL_UNIFORM, synth.AL_UNIFORM)
    ops = 0
    secs = 0.0
    done = 0
    bad = 0
    for li, L in runner_layers:
        per = L.h * L.h * L.cin
        x = synth.counter_codes_host(image * per, per, (cfg, li, synth.T_X), "relu").reshape(1, L.h, L.h, L.cin)
        w = synth.counter_codes_host(0, L.cout * L.k * L.k * L.cin, (cfg, li, synth.T_W),
                                     "uniform").reshape(L.cout, L.k, L.k, L.cin)
        t0 = time.perf_counter()
        acc = oracle.conv2d_direct(x, w, T, L.stride, L.pad, 0)
        r = synth.conv_requant(L)
        codes = oracle.requantize(acc.reshape(-1, L.cout), r.mult, r.shift, r.zp, r.qmin, r.qmax,
                                  bias=np.full(L.cout, r.bias, np.int32), bias_axis=0)
        secs += time.perf_counter() - t0
        ops += 2 * L.cout * L.ho * L.ho * L.k * L.k * L.cin
        done += 1
        if check is not None and li in check:
            g = check[li]
            got = oracle.unpack_codes(g, g.shape[0], L.cout, g.shape[1])
            bad += int((got != codes).sum())
        if secs > budget_s:
            break
    return ops, secs, done, bad


def oracle_all_cores(cfg, runner_layers, images, check):
    """The same oracle (unchanged, single-threaded C) run on every host core at once: one image per
    thread (ctypes releases the GIL), all layers; also compares each image with the GPU codes in
    `check` (layer index -> host codes of the whole local batch, rows image-major).
    Returns (ops, wall seconds, threads, mismatched codes)."""
    from concurrent.futures import ThreadPoolExecutor

    def one(slot_image):
        slot, image = slot_image
        sub = {}
        for li, L in runner_layers:
            rows = L.ho * L.ho
            sub[li] = check[li][slot * rows:(slot + 1) * rows]
        o, _, _, bad = oracle_conv_sample(cfg, runner_layers, image, budget_s=1e9, check=sub)
        return o, bad

    t0 = time.perf_counter()
    with ThreadPoolExecutor(max_workers=len(images)) as ex:
        res = list(ex.map(one, images))
    wall = time.perf_counter() - t0
    return sum(r[0] for r in res), wall, len(images), sum(r[1] for r in res)


# ---------------------------------------------------------------- conv workloads
def run_conv(args, ws, rank, local):
    import synth
    from paper_2304_09049_b200 import dg, netrun
    cfg = {"resnet50": 3, "vgg16": 4}[args.workload]
    batch = args.batch or synth.CONFIG_BATCH[cfg]
    from paper_2304_09049_b200 import shard
    images = list(shard.batch_shard(rank, ws, batch))         # weak scaling: disjoint shards
    torch.cuda.synchronize()
    # weights and biases are prepared once here and synchronised: the step's kernels may read them
    # before their programmatic-dependent-launch wait (dg.h "early_weights")
    dg.set_option("early_weights", 1)
    runner = netrun.NetRunner(cfg, images, "cuda", variant=args.variant)
    nl = len(runner.plans)
    stream = torch.cuda.current_stream()
    # warm-up (untimed): also sets kernel attributes before graph capture
    for _ in range(max(1, args.warmup)):
        runner.step()
    torch.cuda.synchronize()
    # The step graph holds the layer launches back to back: each kernel's prologue overlaps the
    # previous one's tail (programmatic dependent launch).  Per-layer external events inside that
    # graph would break the overlap (measured: 1.58 -> 2.06 ms per ResNet-50 step), so the timed
    # region replays the plain graph and a separate instrumented graph gives the per-layer times.
    graph = torch.cuda.CUDAGraph()
    n0 = dg.kernel_launches()   # native counter of libdg launches (each captured launch counts once)
    with torch.cuda.graph(graph):
        runner.step()
    launches_per_step = dg.kernel_launches() - n0
    gev = [(torch.cuda.Event(enable_timing=True, external=True), torch.cuda.Event(enable_timing=True, external=True))
           for _ in range(nl)]
    graph_ev = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph_ev):
        runner.step(gemm_events=gev)
    for _ in range(args.warmup):
        graph.replay()
        graph_ev.replay()
    torch.cuda.synchronize()

    # ---- timed region
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier(ws)
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        e0.record()
        for _ in range(args.steps):
            graph.replay()
        e1.record()
        torch.cuda.synchronize()
    barrier(ws)
    ms = e0.elapsed_time(e1) / args.steps
    # the outputs the TIMED graph replays wrote, kept before anything else rewrites them (parity leg)
    snap = [p.out.clone() for p in runner.plans]
    # per-layer GEMM times: one instrumented replay after the timed region (layers run unoverlapped)
    graph_ev.replay()
    torch.cuda.synchronize()
    gemm_ms = [a.elapsed_time(b) for a, b in gev]
    replay_equal = all(torch.equal(a, p.out) for a, p in zip(snap, runner.plans))
    ms_max = max_over_ranks(ms, ws)
    ops_step = runner.total_ops
    value = ops_step * ws / (ms_max * 1e-3) / 1e12

    # ---- dominant kernel roofline (tensor pipe, int8 dense peak).  Every launch in the timed step is
    # lut_gemm_ts_kernel (one per layer, back to back on this stream), so its achieved rate over the
    # timed region is the step's ops / the step's event time.
    pk = peaks()
    gemm_total_ms = sum(gemm_ms)
    achieved = ops_step / (ms * 1e-3) / 1e12
    tr = None
    if os.path.exists(TRAFFIC):
        with open(TRAFFIC) as f:
            t = json.load(f).get(args.workload)
            tr = t["bytes_per_launch"] if t else None
    # algorithmic bytes of a GEMM launch: packed input + packed weights + packed output
    alg_bytes = (runner.input_bytes() + runner.weight_bytes() + runner.output_bytes()) / nl
    # per-layer roofline t_roof = max(ops / int8 peak, algorithmic bytes / HBM): the fraction of it
    # the measured GEMM times reach (HBM-bound 1x1 layers count against bandwidth)
    t_roof = 0.0
    for p_ in runner.plans:   # (layers on the FP4 conv kernel against the e2m1 peak, 2 x int8)
        lb = p_.x.numel() + p_.w.numel() + p_.out.numel()
        peak_l = pk["i8_burst"] * (2.0 if p_.w4 is not None else 1.0)
        t_roof += max(p_.ops / (peak_l * 1e12), lb / (pk["hbm_gbs"] * 1e9))
    n_f4 = sum(1 for p_ in runner.plans if p_.w4 is not None)
    frac_layer = t_roof / (ms * 1e-3)
    # per kernel: its share of the step (instrumented per-layer times), the step time that share
    # stands for, its own ops, and the peak of its own pipe (kind::i8 = 2 x bf16, kind::mxf4 = 2 x i8)
    per_kernel = {}
    for name, is_f4, peak_k in (("lut_conv_f4_kernel", True, 2.0 * pk["i8_burst"]),
                                ("lut_gemm_ts_kernel", False, pk["i8_burst"])):
        idx = [i for i, p_ in enumerate(runner.plans) if (p_.w4 is not None) == is_f4]
        if not idx:
            continue
        share = sum(gemm_ms[i] for i in idx) / gemm_total_ms
        ops_k = sum(runner.plans[i].ops for i in idx)
        ach = ops_k / (share * ms * 1e-3) / 1e12
        per_kernel[name] = {"layers": len(idx), "time_share": round(share, 4), "achieved": round(ach, 1),
                            "peak": round(peak_k, 1), "frac": round(ach / peak_k, 4)}
    mixed_peak = ops_step / sum(p_.ops / (pk["i8_burst"] * (2.0 if p_.w4 is not None else 1.0)) for p_ in runner.plans)
    # the top-level fields describe the DOMINANT kernel (largest share of the step): its ops over the
    # step time its share stands for, against the peak of its own pipe; its traffic per launch from
    # the committed ncu launch list; the whole step's figures follow as step_*
    dom = max(per_kernel, key=lambda k: per_kernel[k]["time_share"]) if per_kernel else "lut_gemm_ts_kernel"
    dk = per_kernel.get(dom, {"achieved": achieved, "peak": pk["i8_burst"], "frac": achieved / pk["i8_burst"]})
    dom_f4 = dom == "lut_conv_f4_kernel"
    d_idx = [i for i, p_ in enumerate(runner.plans) if (p_.w4 is not None) == dom_f4]
    d_alg = sum(runner.plans[i].x.numel() + runner.plans[i].w.numel() + runner.plans[i].out.numel() for i in d_idx) / max(1, len(d_idx))
    d_tr = None
    if os.path.exists(TRAFFIC):
        with open(TRAFFIC) as f:
            t = json.load(f).get(args.workload) or {}
            d_tr = (t.get("per_kernel") or {}).get(dom)
    roof = {"bound": "tensor",
            "kernel": (f"lut_conv_f4_kernel (tcgen05 kind::mxf4, {n_f4} of {nl} layers)" if dom_f4 else
                       f"lut_gemm_ts_kernel (tcgen05 kind::i8, A in TMEM, {nl - n_f4} of {nl} layers)"),
            "achieved": dk["achieved"], "peak": dk["peak"], "unit": "TOPS", "frac": dk["frac"],
            "traffic": round(d_tr) if d_tr else None, "alg_bytes_per_launch": round(d_alg),
            "time_share": dk.get("time_share"),
            "peak_src": pk["src"] + (": e2m1 (kind::mxf4) = 2 x int8 = 4 x the measured bf16 burst (nominal 9 / 4.5 / 2.25)"
                                     if dom_f4 else ": int8 = 2 x the measured bf16 burst (nominal 4.5 / 2.25)"),
            "achieved_src": "the kernel's ops / (its share of the step, from per-layer CUDA events in an instrumented "
                            "replay of the step graph, x the timed step time)",
            "step_kernels": "lut_gemm_ts_kernel (tcgen05 kind::i8, A in TMEM)" + (
                f" + lut_conv_f4_kernel (kind::mxf4) on {n_f4} of {nl} layers" if n_f4 else ""),
            "step_achieved": round(achieved, 1), "step_peak_i8": round(pk["i8_burst"], 1),
            "step_frac_vs_i8_peak": round(achieved / pk["i8_burst"], 4),
            "step_frac_vs_sustained_i8_peak": round(achieved / pk["i8_sustained"], 4),
            "step_achieved_src": "sum of the step's GEMM ops / step time over the timed region (CUDA events on the launching stream; the step is only the layers' GEMM kernel launches)",
            "instrumented_gemm_ms_sum": round(gemm_total_ms, 4),
            "frac_vs_layer_roofline": round(frac_layer, 4),
            "i8_mma_ceiling": None,
            "layer_roofline_ms": round(t_roof * 1e3, 4),
            "step_traffic": tr, "step_alg_bytes_per_launch": round(alg_bytes),
            "traffic_src": "profiles/traffic.json (ncu dram__bytes_read+write per launch, profiles/r02_launches_resnet50.csv)",
            "mixed_peak": round(mixed_peak, 1),
            "frac_vs_mixed_peak": round(achieved / mixed_peak, 4),
            "mixed_peak_src": "ops-weighted: every layer at the peak of the pipe it runs on (int8 burst, or 2 x that for kind::mxf4)",
            "per_kernel": per_kernel}

    # ---- end to end through the public C ABI (dg_lut_conv2d) with host buffers
    e2e = None
    if args.e2e_steps > 0:
        h_in = [torch.empty(p.x.shape, dtype=torch.uint8, pin_memory=True) for p in runner.plans]
        h_out = [torch.empty(p.out.shape, dtype=torch.uint8, pin_memory=True) for p in runner.plans]
        for h, p in zip(h_in, runner.plans):
            h.copy_(p.x)
        torch.cuda.synchronize()

        # layer-pipelined: layer i's H2D copy (stream s_in), conv (s_cmp, after its input landed) and
        # D2H copy (s_out, after its conv) overlap the other layers' transfers; PCIe is full duplex,
        # so the input and output streams run concurrently.  A step's inputs are overwritten only
        # after the previous step's convs, its outputs only after the previous step's D2H copies.
        cur = torch.cuda.current_stream()
        s_in, s_cmp, s_out = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
        ev_in = [torch.cuda.Event() for _ in runner.plans]
        ev_cv = [torch.cuda.Event() for _ in runner.plans]

        def e2e_step():
            s_in.wait_stream(s_cmp)
            s_cmp.wait_stream(s_out)
            for i, (h, p) in enumerate(zip(h_in, runner.plans)):
                with torch.cuda.stream(s_in):
                    p.x.copy_(h, non_blocking=True)
                ev_in[i].record(s_in)
            for i, p in enumerate(runner.plans):
                s_cmp.wait_event(ev_in[i])
                runner.conv2d_layer(i, stream=s_cmp)
                ev_cv[i].record(s_cmp)
            for i, (h, p) in enumerate(zip(h_out, runner.plans)):
                s_out.wait_event(ev_cv[i])
                with torch.cuda.stream(s_out):
                    h.copy_(p.out, non_blocking=True)

        e2e_step()
        torch.cuda.synchronize()
        barrier(ws)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(cur)
        s_in.wait_stream(cur)
        for _ in range(args.e2e_steps):
            e2e_step()
        cur.wait_stream(s_out)
        cur.wait_stream(s_cmp)
        b.record(cur)
        torch.cuda.synchronize()
        barrier(ws)
        ems = max_over_ranks(a.elapsed_time(b) / args.e2e_steps, ws)
        e2e = {"value": round(ops_step * ws / (ems * 1e-3) / 1e12, 2), "unit": "TOPS",
               "ms_per_step": round(ems, 3), "h2d_bytes_per_step": runner.input_bytes(),
               "d2h_bytes_per_step": runner.output_bytes(),
               "api": "dg_lut_conv2d (pinned host buffers; per-layer H2D / conv / D2H on three streams)"}

    # ---- parity of the TIMED outputs (snapshot) on sampled images + the CPU oracle baseline
    cpu = None
    parity = None
    if rank == 0 and not args.no_oracle:
        all_layers = synth.CONFIG_LAYERS[cfg]()
        check = {li: t.cpu().numpy() for t, li in zip(snap, runner.layer_ids)}
        del snap
        sel = [(li, all_layers[li]) for li in runner.layer_ids]
        model, ncores = cpu_info()
        # (1) the oracle as it stands, one thread, first local image, every layer
        o_ops, o_s, done, bad1 = oracle_conv_sample(cfg, sel, images[0], budget_s=args.oracle_budget,
                                                    check={li: c[:all_layers[li].ho ** 2] for li, c in check.items()})
        # (2) the same oracle on every host core: one image per core, spread over the local batch
        nimg = max(2, min(ncores, len(images), args.oracle_images))
        slots = sorted(set(int(round(i * (len(images) - 1) / (nimg - 1))) for i in range(nimg)))
        a_ops, a_s, a_thr, bad2 = oracle_all_cores(cfg, sel, [(s_, images[s_]) for s_ in slots], check)
        parity = {"of": "outputs of the timed graph replays (snapshot before any other replay)",
                  "images": [images[s_] for s_ in slots], "layers_checked": len(sel),
                  "mismatched_codes": bad1 + bad2, "instrumented_replay_equal": replay_equal,
                  "status": "bit-exact" if bad1 + bad2 == 0 and replay_equal else "MISMATCH"}
        if ws == 1:
            cpu = {"value": o_ops / o_s / 1e12, "unit": "TOPS", "cores": 1, "kind": "oracle",
                   "cpu_model": model, "host_cores": ncores,
                   "sample": f"oracle/oracle.c conv2d_direct+requantize, image {images[0]}, first {done} of {nl} "
                             f"layers ({o_ops / 1e9:.2f} GOP in {o_s:.1f} s), single thread",
                   "all_cores": {"value": a_ops / a_s / 1e12, "unit": "TOPS", "cores": a_thr,
                                 "sample": f"the same oracle on {a_thr} threads, one image each (images "
                                           f"{[images[s_] for s_ in slots][:4]}...), all {nl} layers: "
                                           f"{a_ops / 1e9:.1f} GOP in {a_s:.1f} s wall"}}

    clocks = clk.summary()
    ceil = i8_mma_ceiling(clocks["sm_mhz"])
    roof["i8_mma_ceiling"] = round(ceil, 1)
    roof["step_frac_vs_i8_mma_ceiling"] = round(achieved / ceil, 4)
    roof["i8_mma_ceiling_src"] = ("tools/mma_bench.cu: 64 SM cycles per 128x128x32 kind::i8 MMA (16384 ops/clk/SM) "
                                  "x 148 SMs x the median SM clock of the timed region")
    gemm_big = None
    if args.gemm_n > 0:   # config 5 (BJ configs[4]) in the same process: the headline GEMM
        gemm_big = gemm_line(args, ws, rank, local, args.gemm_n, levels="learned", variant="auto")
    if rank == 0:
        line = {"metric": METRIC, "value": round(value, 2), "unit": "TOPS", "n_gpus": ws,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_max, 4),
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int8",
                "data": "synthetic (seeded counter-based 2-bit codes; ReLU-skewed activations)",
                "config": {"workload": f"{args.workload}_b{batch}_lut_conv (BASELINE configs[{cfg - 1}])",
                           "layers": nl, "batch_per_gpu": batch, "global_batch": batch * ws,
                           "ops_per_step_per_gpu": ops_step, "variant": args.variant,
                           "l2": f"inputs larger than L2: {runner.input_bytes() / 1e9:.2f} GB of per-layer "
                                 "independent packed inputs per step per GPU (126 MB L2)",
                           "parallelism": f"dp{ws} (batch shards, no collective in the step)"},
                "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": launches_per_step * args.steps, "clocks": clocks,
                "parity": parity, "gemm_ms_per_layer": [round(x, 4) for x in gemm_ms],
                "kernel_per_layer": [p.kernel for p in runner.plans]}
        if gemm_big is not None:
            line[f"gemm{args.gemm_n}"] = gemm_big
        print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- config 2: ResNet-18 b1 chain
def run_resnet18(args, ws, rank, local):
    """BJ configs[1]: the 19 LUT convs of ResNet-18 at batch 1, chained with int32 residual adds.
    Latency-bound, so the whole chain is one CUDA graph; every rank runs an independent replica
    (replicas only: batch 1 does not shard)."""
    from paper_2304_09049_b200 import dg, netrun
    r = netrun.ResNet18Runner("cuda", variant=args.variant, batch=args.batch or 1)
    for _ in range(max(1, args.warmup)):
        r.step()
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    n0 = dg.kernel_launches()
    with torch.cuda.graph(graph):
        r.step()
    launches_per_step = dg.kernel_launches() - n0   # (split-K convs add a reduce kernel)
    for _ in range(args.warmup):
        graph.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier(ws)
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        e0.record()
        for _ in range(args.steps):
            graph.replay()
        e1.record()
        torch.cuda.synchronize()
    barrier(ws)
    ms = max_over_ranks(e0.elapsed_time(e1) / args.steps, ws)
    value = r.total_ops * ws / (ms * 1e-3) / 1e12
    if rank == 0:
        pk = peaks()
        line = {"metric": METRIC, "value": round(value, 2), "unit": "TOPS", "n_gpus": ws, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": round(ms, 4), "us_per_image": round(ms * 1e3 / r.B, 2),
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int8",
                "data": "synthetic (seeded counter-based 2-bit codes; calibrated requant, synth_data/)",
                "config": {"workload": f"resnet18_b{r.B}_chain (BASELINE configs[1])", "layers": len(r.layers),
                           "parallelism": f"{ws} independent replicas"},
                "roofline": {"bound": "latency", "achieved": round(value / ws, 2), "peak": round(pk["i8_burst"], 1),
                             "unit": "TOPS", "frac": round(value / ws / pk["i8_burst"], 5)},
                "gpu_launches": launches_per_step * args.steps, "clocks": clk.summary()}
        print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- config 5: square LUT-GEMM
def gemm_line(args, ws, rank, local, n, levels="learned", variant="auto"):
    """BJ configs[4]: C[n][n] = sum_k T[(W<<2)|A] with learned-style int16 levels (Q17), int32 out.
    Output channels (rows of W / C) are split across ranks; the int32 row blocks are all-gathered
    over NCCL so every rank holds C; --fused-gather stores every tile into all
    ranks' C from the GEMM epilogue instead (P2P, symmetric memory).  Returns rank 0's JSON dict
    (None elsewhere): compute-only and end-to-end TOPS, roofline, clocks, exact parity of the
    WHOLE gathered C (Freivalds) + sampled rows from every rank's block."""
    import synth
    from paper_2304_09049_b200 import dg, shard
    r0, r1 = shard.row_shard(rank, ws, n)
    m_loc = r1 - r0
    f4 = variant == "f4"
    onehot = variant == "onehot"
    T_any = None
    if onehot:   # an arbitrary (non-product) int8 table, seeded: the one-hot K' = 4K tensor-core path
        T_any = np.random.default_rng(synth.MASTER_SEED + 5).integers(-127, 128, 16).astype(np.int32)
        lut = dg.lut_from_table(T_any, 8)
        wl = al = None
    elif levels == "uniform" or f4:   # config-1 levels (the FP4 path needs e2m1-representable levels)
        wl, al = list(synth.WL_UNIFORM), list(synth.AL_UNIFORM)
        lut = dg.build_lut(wl, al, 8)
    else:
        wl, al = synth.learned_levels(5, 0, synth.T_LEVELS)
        lut = dg.build_lut(wl, al, 16)
    dev = "cuda"
    ld = dg.packed_ld(n)
    # codes: W rows [rank*m_loc, (rank+1)*m_loc), A^T all n rows; counter generator (same on CPU)
    w_codes = synth.counter_codes(rank * m_loc * n, m_loc * n, (5, n, synth.T_W), "uniform", dev).view(m_loc, n)
    w = dg.pack_weights(w_codes)
    del w_codes
    at = torch.empty((n, ld), dtype=torch.uint8, device=dev)
    chunk = max(1, (1 << 26) // n)
    for q0 in range(0, n, chunk):
        q1 = min(n, q0 + chunk)
        c = synth.counter_codes(q0 * n, (q1 - q0) * n, (5, n, synth.T_A), "uniform", dev).view(q1 - q0, n)
        dg.pack_codes(c, out=at[q0:q1])
    if f4:   # block-scaled FP4 path: the weights are expanded once to e2m1, activations stay packed
        w4 = dg.expand_operand_f4(w, n, wl)
        at8 = None
    elif onehot:   # both operands expanded once: one-hot weight codes, int8 table columns
        w1h = dg.expand_onehot(w, n)
        atc = dg.expand_tcols(at, n, lut)
        at8 = None
    else:
        at8 = dg.expand_operand(at, n, al)          # offline expansion of the second operand
    peer = None
    if ws > 1 and args.fused_gather and not f4 and not onehot:
        try:
            peer = shard.PeerRows((n, n), torch.int32, dev, rank, ws, rank * m_loc)
        except Exception as e:  # (no P2P / symmetric memory on this node)
            print(f"[bench] fused all-gather unavailable ({type(e).__name__}: {e}); using NCCL", file=sys.stderr)
    if peer is not None:
        c_full = peer.full
        c_loc = c_full[rank * m_loc:(rank + 1) * m_loc]
    else:
        c_loc = torch.empty((m_loc, n), dtype=torch.int32, device=dev)
        c_full = torch.empty((n, n), dtype=torch.int32, device=dev) if ws > 1 else c_loc
    ops_total = 2 * n * n * n

    def gemm():
        if f4:
            dg.lut_gemm_f4(w4, at, m_loc, n, n, lut, out=c_loc)
        elif onehot:
            dg.lut_gemm_onehot(w1h, atc, m_loc, n, n, lut, out=c_loc)
        elif peer is not None:
            dg.lut_gemm_prepared_allgather(w, at8, m_loc, n, n, lut, c_loc, peer.peers)
        else:
            dg.lut_gemm_prepared(w, at8, m_loc, n, n, lut, out=c_loc)

    def gather():
        if peer is not None:
            peer.barrier()
        elif ws > 1:
            shard.gather_rows(c_loc, ws, out=c_full)

    for _ in range(max(3, args.warmup)):
        gemm()
        gather()
    torch.cuda.synchronize()
    kernel = dg.last_kernel()
    # L2 is flushed between steps by the 1 GiB int32 output of n=16384 itself; for smaller n a
    # 256 MB scratch write is issued between steps (outside the events).
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev) if n < 16384 else None
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    g1 = torch.cuda.Event(enable_timing=True)
    t_comp = 0.0
    t_all = 0.0
    steps = max(3, args.gemm_steps if args.workload != "gemm" else args.steps)
    barrier(ws)
    torch.cuda.synchronize()
    n0 = dg.kernel_launches()
    with ClockSampler(local) as clk:
        for _ in range(steps):
            if flush is not None:
                flush.zero_()
            barrier(ws)
            e0.record()
            gemm()
            e1.record()
            gather()
            g1.record()
            torch.cuda.synchronize()
            t_comp += e0.elapsed_time(e1)
            t_all += e0.elapsed_time(g1)
    launches = dg.kernel_launches() - n0
    barrier(ws)
    ms_comp = max_over_ranks(t_comp / steps, ws)
    ms_all = max_over_ranks(t_all / steps, ws)
    pk = peaks()
    value = ops_total / (ms_all * 1e-3) / 1e12
    comp_tops = ops_total / (ms_comp * 1e-3) / 1e12
    per_gpu = (2 * m_loc * n * n) / (t_comp / steps * 1e-3) / 1e12
    # parity (rank 0): exact Freivalds over the WHOLE gathered C (every rank's rows) + the first and
    # last row of every rank's block against the oracle
    parity = None
    if not args.no_oracle and rank == 0:
        import oracle
        C = c_full.cpu().numpy()
        Wc = synth.counter_codes_host(0, n * n, (5, n, synth.T_W), "uniform").reshape(n, n)
        Atc = synth.counter_codes_host(0, n * n, (5, n, synth.T_A), "uniform").reshape(n, n)
        T = T_any if onehot else oracle.build_lut16(wl, al)
        t0 = time.perf_counter()
        bad = oracle.freivalds_rows(Wc, Atc, C, T, trials=1)
        rows = sorted(set([r_ * m_loc for r_ in range(ws)] + [r_ * m_loc + m_loc - 1 for r_ in range(ws)]))
        ref = oracle.lut_gemm(Wc[rows], np.ascontiguousarray(Atc.T), T)
        parity = {"of": f"the whole gathered C ({ws} rank block(s))", "freivalds_bad_rows": bad,
                  "sampled_rows": rows[:16], "sampled_rows_equal": bool(np.array_equal(ref, C[rows])),
                  "status": "bit-exact" if bad == 0 and np.array_equal(ref, C[rows]) else "MISMATCH",
                  "oracle_s": round(time.perf_counter() - t0, 1)}
    if rank != 0:
        return None
    clocks = clk.summary()
    alg_bytes = m_loc * ld + n * ld + 4 * m_loc * n
    scale = 2.0 if f4 else (0.25 if onehot else 1.0)   # onehot: 4K MMA terms per K lookups
    peak = pk["i8_burst"] * scale
    peak_s = pk["i8_sustained"] * scale
    ceil = i8_mma_ceiling(clocks["sm_mhz"]) * scale
    uni = wl is not None and list(wl) == list(synth.WL_UNIFORM)
    return {"metric": METRIC, "value": round(value, 2), "unit": "TOPS", "n_gpus": ws, "steps": steps,
            "warmup": args.warmup, "ms_per_step": round(ms_all, 4), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "e2m1" if f4 else "int8",
            "data": ("synthetic (seeded counter-based 2-bit codes; seeded random non-product int8 table)" if onehot else
                     "synthetic (seeded counter-based 2-bit codes; config-1 levels wl={-2..1}, al={0..3})" if uni else
                     "synthetic (seeded counter-based 2-bit codes; learned-style int16 levels, Q17)"),
            "config": {"workload": (f"square_gemm_n{n}, config-1 levels, FP4 path (SURVEY 8(f) rank 2)" if f4 else
                                    f"square_gemm_n{n}, non-product int8 table, one-hot K'=4K tensor-core path (SURVEY 8(f) rank 3)" if onehot else
                                    f"square_gemm_n{n} (BASELINE configs[4])" + (", config-1 levels" if uni else "")),
                       "n": n, "kernel": kernel,
                       "split": (f"output channels / {ws}; " + ("fused all-gather: epilogue stores every tile into all ranks' C (NVLink P2P, symmetric memory)" if peer is not None else "NCCL all_gather_into_tensor of int32 rows")) if ws > 1 else "none",
                       "l2": "1 GiB int32 output per step (> L2)" if flush is None else "256 MB L2 flush between steps"},
            "compute_only": {"value": round(comp_tops, 2), "ms": round(ms_comp, 4), "per_gpu_tops": round(per_gpu, 2)},
            "roofline": {"bound": "tensor",
                         "kernel": ("lut_gemm_f4_kernel (tcgen05 kind::mxf4, e2m1, SS)" if f4 else
                                    "lut_gemm_ts_kernel (tcgen05 kind::i8, A in TMEM)"),
                         "achieved": round(per_gpu, 1), "peak": round(peak, 1), "unit": "TOPS",
                         "frac": round(per_gpu / peak, 4),
                         "frac_vs_sustained_peak": round(per_gpu / peak_s, 4),
                         "i8_mma_ceiling": round(ceil, 1), "frac_vs_i8_mma_ceiling": round(per_gpu / ceil, 4),
                         "peak_src": pk["src"] + (": e2m1 dense = 4 x bf16 burst (nominal 9/2.25)" if f4 else
                                                  ": int8 = 2 x bf16 burst / 4 (the one-hot form runs 4K int8 MACs per K lookups)" if onehot else
                                                  ": int8 = 2 x bf16 burst (kernel timed alone)"),
                         "alg_bytes_per_launch": alg_bytes, "traffic": None},
            "gpu_launches": launches, "clocks": clocks, "parity": parity}


def run_gemm(args, ws, rank, local):
    line = gemm_line(args, ws, rank, local, args.n, levels=args.levels, variant=args.variant)
    if line is not None:
        print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- reference arm (the oracle)
def run_reference(args, ws, rank):
    """--impl reference: the oracle as it stands, on the host cores, on the same config /
    metric / unit.  Each step is a bounded sample (one image through a rotating subset of
    layers).  Under torchrun only rank 0 runs; the others exit 0 without work."""
    if rank != 0:
        return
    import synth
    cfg = {"resnet50": 3, "vgg16": 4}.get(args.workload, 3)
    layers = synth.CONFIG_LAYERS[cfg]()
    per_step = max(1, len(layers) // 13)
    ops_t, s_t = 0, 0.0
    li = 0
    for st in range(args.warmup + args.steps):
        sel = []
        for _ in range(per_step):
            sel.append((li % len(layers), layers[li % len(layers)]))
            li += 1
        o, s, _, _ = oracle_conv_sample(cfg, sel, 0, budget_s=1e9)
        if st >= args.warmup:
            ops_t += o
            s_t += s
    v = ops_t / s_t / 1e12
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "TOPS", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": s_t * 1e3 / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64",
            "data": "synthetic", "config": {"workload": f"{args.workload} (oracle sample)"},
            "cpu_baseline": {"value": v, "unit": "TOPS", "cores": 1, "kind": "oracle",
                             "sample": f"{per_step} layer(s) of image 0 per step, rotating over the {len(layers)} layers"},
            "e2e": {"value": v, "unit": "TOPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="resnet50", choices=["resnet50", "vgg16", "gemm", "resnet18"])
    ap.add_argument("--n", type=int, default=16384, help="config 5 GEMM size (4096 / 8192 / 16384)")
    ap.add_argument("--variant", default="auto", choices=["auto", "cc", "tc", "f4", "onehot"],
                    help="gemm workload: f4 = block-scaled FP4 path (config-1 levels); onehot = any int8 table (K' = 4K)")
    ap.add_argument("--levels", default="learned", choices=["learned", "uniform"],
                    help="gemm workload: learned int16 levels (BJ configs[4]) or config-1 levels")
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--oracle-budget", type=float, default=20.0)
    ap.add_argument("--no-oracle", action="store_true")
    ap.add_argument("--fused-gather", action="store_true",
                    help="config 5 at N > 1: all-gather fused into the GEMM epilogue over P2P (default: NCCL all_gather)")
    ap.add_argument("--gemm-n", type=int, default=16384,
                    help="conv workloads: also time config 5 at this n in the same run (0 = skip)")
    ap.add_argument("--gemm-steps", type=int, default=10)
    ap.add_argument("--oracle-images", type=int, default=64, help="images checked by the all-core oracle leg")
    args = ap.parse_args()
    ws, rank, local = dist_env()
    if os.environ.get("DG_OPTS"):   # ablation hook: "name=value,name=value" (dg_set_option)
        from paper_2304_09049_b200 import dg
        for kv in os.environ["DG_OPTS"].split(","):
            k, v = kv.split("=")
            dg.set_option(k, int(v))
    if args.impl == "reference":
        return run_reference(args, ws, rank)
    torch.cuda.set_device(local)
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    try:
        if args.workload == "gemm":
            run_gemm(args, ws, rank, local)
        elif args.workload == "resnet18":
            run_resnet18(args, ws, rank, local)
        else:
            run_conv(args, ws, rank, local)
    finally:
        if ws > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
