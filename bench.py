#!/usr/bin/env python
"""Benchmark of the MLFMA near-field P2P operator on B200 (BASELINE.json metric:
P2P pair-interactions/s; roofline fraction).

One *step* = one apply of the whole hot path (SURVEY.md §8(a) apply rows:
[halo weight exchange] -> P2P kernel) over each config of the workload, with
inputs resident in HBM.  Default workload = BASELINE.json configs[3], the
configuration the metric is quoted on at 1/2/4/8 B200: the 2e7-point
surface-like cloud (a 1250 x 1000-box plate at L = 12, 16 points per box),
TILED layout (redundant only on the tile ring), fp32 (the headline), Morton
plan order; the same step in fp64 is the "fp64" field, the NR and R layouts
are reported under "extras".

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]
  torchrun --nproc-per-node N bench.py --gpus N ...   (strong scaling: the same global problem
                                                       Morton-range sharded, NCCL halo exchange)

Timing: W warm-up steps, then K steps timed with CUDA events on the apply
stream, L2 flushed (256 MiB write) between steps, barrier + synchronize on
both sides, max over ranks.  Clocks are sampled with NVML during the timed
region.  The CPU baseline is the fp64 oracle (oracle/, test infrastructure)
on a bounded sample of the same workload, rank 0 at N = 1 only.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2403_01596_b200 import workloads as W  # noqa: E402

WORKLOADS = {
    "density_1e6": ["d16_1e6", "d32_1e6", "d64_1e6"],           # configs[1]
    "lowdensity_1e7": ["lowd025_1e7", "lowd1_1e7", "lowd2_1e7", "lowd4_1e7"],  # configs[2]
    "surface_2e7": ["surf_2e7"],                                # configs[3] (headline, default)
    "d32_7e7": ["d32_7e7"],                                     # configs[4]
    "tiny": ["tiny"],                                           # configs[0]
    "helmholtz_1e6": ["d16_1e6", "d4_1e6"],                     # NEXT-3: 2D Helmholtz, leaf = lambda/4
    "contour_2e5": ["contour_2e5"],                             # NEXT-4: curve cloud, Laplace
    "contour_helmholtz": ["contour_1e5"],                       # NEXT-4: curve cloud, Helmholtz, leaf = lambda/4
    "cube3d_1e6": ["cube3d_1e6"],                               # NEXT-3: 3D Laplace, 16 per box
    "cube3d_helmholtz": ["cube3d_1e6"],                         # NEXT-3: 3D Helmholtz, leaf = lambda/4
}
DEFAULT_KERNEL = {"helmholtz_1e6": "helmholtz", "contour_helmholtz": "helmholtz", "cube3d_1e6": "laplace3d",
                  "cube3d_helmholtz": "helmholtz3d"}
MUFU_PER_PAIR_3D = {"laplace3d": 1, "helmholtz3d": 3}  # RSQ; RSQ + SIN + COS
METRIC = "P2P pair-interactions/s"
SM_COUNT = 148
PEAKS_JSON = os.path.join(ROOT, "profiles", "r02_peaks.json")  # tools/peaks.py on a B200 (libp2p_peaks.so)
FP64_DP_OPS_PER_PAIR = 14  # r^2 + guard + accumulate (6) + the table-driven log (8)


def _measured_peaks():
    """MUFU.LG2 and DFMA rates per clock per SM measured by tools/peaks.py (committed JSON); the
    nominal 16 lg2 / 64 DFMA per clk per SM (B200_PROFILING.md) if the file is absent."""
    try:
        d = json.load(open(PEAKS_JSON))
        return (d["mufu_lg2"]["per_clk_per_sm"], d["dfma"]["per_clk_per_sm"] / 2.0,
                f"profiles/r02_peaks.json (measured {d['when'][:10]}: {d['mufu_lg2']['per_clk_per_sm']:.2f} "
                f"lg2/clk/SM, {d['dfma']['per_clk_per_sm'] / 2:.2f} DFMA/clk/SM)")
    except Exception:
        return 16.0, 64.0, "nominal 16 lg2 / 64 DFMA per clk per SM (profiles/r02_peaks.json absent)"


MUFU_LG2_PER_CLK_PER_SM, DFMA_PER_CLK_PER_SM, PEAK_BASIS = _measured_peaks()
try:  # FP32 FMA lanes per clk per SM (FFMA2 = 2 FMA per lane-instruction; peaks.json counts 4 FLOP)
    FFMA_PER_CLK_PER_SM = json.load(open(PEAKS_JSON))["ffma2"]["per_clk_per_sm"] / 2.0
except Exception:
    FFMA_PER_CLK_PER_SM = 128.0
# 2D Helmholtz, per pair on the series branch (every pair of the kappa h = pi/2 workload):
# fp32: r^2 4, z 1, two degree-10 Horner chains 20, ln 1 (+ MUFU), Y 2, complex multiply-add 4
# fp64: r^2 4, z 1, two degree-18 chains 36, the table log 8, ln 1, Y 2, complex multiply-add 4
HELM_OPS_PER_PAIR = {"fp32": 32, "fp64": 56}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="surface_2e7", choices=sorted(WORKLOADS))
    ap.add_argument("--layout", default="tiled", choices=["nr", "r", "tiled"])
    ap.add_argument("--precision", default="fp32", choices=["fp32", "fp64"])
    ap.add_argument("--kind", default="iid", choices=["iid", "stratified"])
    ap.add_argument("--scaling", default="strong", choices=["weak", "strong"],
                    help="N > 1: strong = the same global problem Morton-range split N ways (SURVEY §8(d) "
                         "E_P = T_1 / (P T_P)); weak = each config's plate widened N x (same points per box)")
    ap.add_argument("--no-extras", action="store_true", help="skip the R / fp64 detail lines")
    ap.add_argument("--build", choices=["device", "host"], default="device",
                    help="N = 1 plans: built on the GPU (p2p_plan_create_device) or by the host builder")
    ap.add_argument("--exchange", choices=["auto", "sync", "nccl", "peer"], default="auto",
                    help="N > 1 halo exchange: sync = one-sided peer-memory reads ordered by device-side "
                         "signals (p2p_apply_peer_sync; CUDA-graph captured); nccl = torch.distributed "
                         "all_to_all; peer = peer-memory reads with host barriers; auto (default) = sync or "
                         "nccl, whichever ran the faster step (max over ranks)")
    ap.add_argument("--no-graph", action="store_true", help="N > 1 sync mode: launch eagerly, no CUDA graph")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true", help="skip the host-buffer e2e leg (quick A/B runs)")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="oracle sample budget")
    ap.add_argument("--profile", action="store_true", help="short run for ncu (no extras/baseline)")
    ap.add_argument("--configs", default="", help="comma list of config names overriding --workload")
    ap.add_argument("--tile", type=int, default=-1, help="force CTA tile side 2^tile (default: plan's choice)")
    ap.add_argument("--kernel", default=None, choices=["laplace", "helmholtz", "laplace3d", "helmholtz3d"],
                    help="kernel function (default: helmholtz for the helmholtz_1e6 workload, else laplace)")
    ap.add_argument("--kh", type=float, default=math.pi / 2,
                    help="helmholtz: kappa * leaf box side (pi/2 = a quarter-wavelength box)")
    a = ap.parse_args()
    if a.kernel is None:
        a.kernel = DEFAULT_KERNEL.get(a.workload, "laplace")
    if a.kernel == "helmholtz":
        a.layout = "tiled"
        a.no_extras = True
    if a.kernel.endswith("3d"):  # the box-per-CTA NR path, host plan build
        a.layout = "nr"
        a.no_extras = True
        a.build = "host"
    return a


def _kernel_kw(args, cfg):
    """Plan keywords of the kernel function (Helmholtz: kappa from the leaf box side)."""
    if args.kernel == "laplace":
        return {}
    kw = {"kernel": args.kernel}
    if args.kernel.startswith("helmholtz"):
        kw["wavenumber"] = args.kh * (1 << (cfg.level - 1))
    return kw


def _weights(args, cfg, q):
    return W.weights_complex(cfg.n, cfg.seed) if args.kernel.startswith("helmholtz") else q


# ---------------------------------------------------------------- clocks
class ClockSampler:
    """NVML sampling of SM clock and throttle reasons during the timed region."""

    REASONS = {
        "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4, "hw_slowdown": 0x8,
        "sync_boost": 0x10, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
        "hw_power_brake_slowdown": 0x80, "display_clock_setting": 0x100,
    }

    def __init__(self, device: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self._nv = None

    def _run(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for name, bit in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self._nv:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._nv:
            self._t.join()

    def summary(self):
        med = float(np.median(self.samples)) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


def _hbm_peak():
    """HBM peak for the roofline: MEASURED_PEAKS.json (driver-written copy bandwidth), else the
    B200_PROFILING.md fallback."""
    try:
        with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "MEASURED_PEAKS.json")) as f:
            v = float(json.load(f)["hbm_gbs"])
        return v, f"MEASURED_PEAKS.json hbm_gbs ({v:.0f} GB/s, copy read+write)"
    except Exception:
        return 7000.0, "fallback 7.0 TB/s (B200_PROFILING.md; MEASURED_PEAKS.json absent)"


# ---------------------------------------------------------------- CPU baseline (oracle)
def cpu_baseline(cfg_names, kind, budget_s, seed_stream=0, kernel="laplace", kh=math.pi / 2):
    """The fp64 oracle as it stands (never tuned), on a bounded, seeded sample of
    the targets of each config, timed on this host's cores."""
    import oracle
    nthreads = oracle.num_threads()
    probs = [(W.CONFIGS[c], *W.make_problem(c, kind=kind)) for c in cfg_names]
    rng = np.random.default_rng(seed_stream)

    def run(cfg, s, t, q, frac):
        sel = np.sort(rng.choice(len(t), max(1, int(frac * len(t))), replace=False))
        tic = time.perf_counter()
        if kernel == "helmholtz":
            _, p = oracle.direct_helmholtz(s, W.weights_complex(cfg.n, cfg.seed), t, cfg.level,
                                           kh * (1 << (cfg.level - 1)), targets=sel)
        elif kernel == "laplace3d":
            _, p = oracle.direct_3d(s, q, t, cfg.level, targets=sel)
        elif kernel == "helmholtz3d":
            _, p = oracle.direct_3d(s, W.weights_complex(cfg.n, cfg.seed), t, cfg.level, "helmholtz",
                                    kh * (1 << (cfg.level - 1)), targets=sel)
        else:
            _, p = oracle.direct(s, q, t, cfg.level, targets=sel)
        return p, time.perf_counter() - tic

    # per config: a 5% probe, then a sample sized to this config's share of the budget
    pairs, secs, fracs = 0, 0.0, []
    share = budget_s / len(probs)
    for cfg, s, t, q in probs:
        p, dt = run(cfg, s, t, q, 0.05)
        f = min(1.0, 0.05 * share / max(dt, 1e-3))
        p, dt = run(cfg, s, t, q, f)
        pairs += p
        secs += dt
        fracs.append(f)
    return {"value": pairs / secs, "unit": "pair-interactions/s", "cores": nthreads, "kind": "oracle",
            "sample": f"{100 * min(fracs):.2f}-{100 * max(fracs):.2f}% of the targets of each of "
                      f"{','.join(cfg_names)} (seeded); fp64 {kernel} direct sum incl. source bucketing; "
                      f"{pairs} pairs in {secs:.1f} s",
            "pairs": pairs, "seconds": secs}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    names = WORKLOADS[args.workload]
    per_step = max(1.0, 150.0 / max(1, args.steps + args.warmup))
    kk = dict(kernel=args.kernel, kh=args.kh)
    for _ in range(args.warmup):
        cpu_baseline(names, args.kind, per_step / 4, **kk)
    vals, pairs, secs = [], 0, 0.0
    last = None
    for k in range(args.steps):
        last = cpu_baseline(names, args.kind, per_step, seed_stream=k + 1, **kk)
        pairs += last["pairs"]
        secs += last["seconds"]
    v = pairs / secs
    cfg = {"workload": args.workload, "configs": names, "layout": "oracle", "kind": args.kind, "kernel": args.kernel}
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": "pair-interactions/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": secs / args.steps * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded SplitMix64 plates, SURVEY.md §8(d))", "config": cfg,
        "cpu_baseline": {"value": v, "unit": "pair-interactions/s", "cores": last["cores"], "kind": "oracle",
                         "sample": last["sample"]},
        "e2e": {"value": v, "unit": "pair-interactions/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))
    return 0


# ---------------------------------------------------------------- GPU path
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist
    from paper_2403_01596_b200 import p2p

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # More ranks than visible GPUs (a 1-GPU test box): ranks share devices and the
    # halo exchange is staged through the host over gloo (test mode, flagged in the JSON).
    shared = world > max(1, torch.cuda.device_count())
    local = local % max(1, torch.cuda.device_count())
    if world > 1:
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream(dev)
    names = args.configs.split(",") if args.configs else WORKLOADS[args.workload]

    # ---- plans (host build + upload; not timed)
    from paper_2403_01596_b200.dist import DistributedP2P
    jobs = []
    weak = world > 1 and args.scaling == "weak"
    for name in names:
        cfg = W.widened(W.CONFIGS[name], world) if weak else W.CONFIGS[name]
        name = cfg.name
        kw = dict(level=cfg.level, layout=args.layout, precision=args.precision, tile_log2=args.tile,
                  **_kernel_kw(args, cfg))
        if world == 1:
            src, tgt, q = W.make_problem(cfg, kind=args.kind)
            q = _weights(args, cfg, q)
            if args.build == "device" and args.layout in ("nr", "tiled"):  # built on the GPU (NEXT-2)
                pl = p2p.Plan(torch.as_tensor(src, device=dev), torch.as_tensor(tgt, device=dev), device=local,
                              build="device", **kw)
            else:
                pl = p2p.Plan(src, tgt, device=local, **kw)
            job = {"name": name, "cfg": cfg, "plan": pl, "info": pl.info, "q_user": q,
                   "q": torch.as_tensor(q[pl.export("src_perm")], dtype=pl.torch_dtype, device=dev)}
        else:  # this rank generates only its share; the plan comes from the ranks' own points
            s_xy, t_xy, sid, tid = W.problem_share(cfg, rank, world, kind=args.kind)
            kw.pop("level")
            dp = DistributedP2P.from_local(s_xy, t_xy, sid, tid, level=cfg.level, device=local, host_staged=shared,
                                           **kw)
            pl = dp.plan
            oid = dp.owned_source_ids()
            qo = (W.weights_complex(cfg.n, cfg.seed, index=oid) if args.kernel.startswith("helmholtz")
                  else W.weights(cfg.n, cfg.seed, index=oid))
            job = {"name": name, "cfg": cfg, "plan": pl, "dp": dp, "info": pl.info,
                   "q_owned": torch.as_tensor(qo, dtype=pl.torch_dtype, device=dev)}
        job["out"] = torch.empty(max(1, job["info"]["n_tgt_local"]), dtype=pl.torch_dtype, device=dev)
        jobs.append(job)
    pairs_step = sum(j["info"]["pairs_global"] for j in jobs)
    pairs_local = sum(j["info"]["pairs"] for j in jobs)

    comm = torch.cuda.Stream(dev) if world > 1 else None
    mode = "single"

    def enqueue(j, cur, ready=None):
        """one config's apply on stream handle `cur` (the current stream: graph-capture safe)"""
        if mode == "single":
            p2p.p2p_apply(j["plan"].handle, j["q"].data_ptr(), j["out"].data_ptr(), p2p.P2P_ORDER_PLAN, 0, cur)
        elif mode == "sync":  # halo pulled from the owners' memory, device-side signals
            j["dp"].apply_sync(j["q_owned"], j["out"], stream=cur)
        elif mode == "peer":  # halo read from the owners' memory (host barriers inside)
            j["dp"].apply_peer(j["q_owned"], j["out"], stream=cur)
        else:
            j["dp"].apply(j["q_owned"], j["out"], stream=cur, halo_ready=ready)

    def step(kev_row=None):
        cur = torch.cuda.current_stream(dev)
        ready = [None] * len(jobs)
        if mode == "nccl":  # all halo exchanges first on the comm stream: config i's overlaps kernel i-1
            comm.wait_stream(cur)
            ready = [j["dp"].exchange_async(j["q_owned"], comm) for j in jobs]
        for i, j in enumerate(jobs):
            if kev_row is not None:
                kev_row[i][0].record(cur)
            enqueue(j, cur.cuda_stream, ready[i])
            if kev_row is not None:
                kev_row[i][1].record(cur)

    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], device="cpu" if shared else dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def prepare(m):
        """warm up exchange mode m; N > 1 sync: capture the whole step (every config's publish /
        pull / interior / boundary kernels) in a CUDA graph -> one graph launch per step"""
        nonlocal mode
        mode = m
        if m == "sync":
            for j in jobs:
                j["dp"].enable_sync()
        for _ in range(max(3, args.warmup)):
            step()
        barrier()
        g = None
        if m == "sync" and not args.no_graph:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                step()
            barrier()
            g.replay()  # one untimed replay (every rank the same count: the epochs stay aligned)
            barrier()
        return g

    # N > 1, --exchange auto: both exchanges, 5 untimed-for-the-record steps each, the faster
    # (max over ranks, so every rank decides alike) is the one timed below
    def all_ok(ok):  # every rank reaches this with its local verdict: a collective decision
        if world == 1:
            return ok
        t = torch.tensor([1 if ok else 0], device="cpu" if shared else dev, dtype=torch.int32)
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        return bool(t.item())

    def sync_ready():
        """Map the peers' buffers (one object all-gather, then local IPC opens) and agree on the
        outcome before any further collective, so a rank that cannot map a peer makes every rank
        fall back to the NCCL exchange instead of diverging."""
        ok = True
        try:
            for j in jobs:
                j["dp"].enable_sync()
        except Exception as e:  # noqa: BLE001 -- reported in the JSON line, decided collectively
            ok = False
            print(f"sync exchange unavailable on rank {rank}: {e}", file=sys.stderr)
        return all_ok(ok)

    autotune = None
    if world > 1 and args.exchange == "auto":
        autotune = {}
        for m in ("sync", "nccl"):
            if m == "sync" and not sync_ready():
                autotune[m] = None
                continue
            g = prepare(m)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            barrier()
            e0.record(stream)
            for _ in range(5):
                g.replay() if g is not None else step()
            e1.record(stream)
            barrier()
            ok = True
            if m == "sync":  # a device-side wait that gave up (20 s) disqualifies the mode everywhere
                try:
                    for j in jobs:
                        j["dp"].check()
                except Exception:  # noqa: BLE001
                    ok = False
            ms_m = max_over_ranks(e0.elapsed_time(e1) / 5)
            autotune[m] = ms_m if all_ok(ok) else None
        chosen = min((m for m in autotune if autotune[m] is not None), key=autotune.get)
    else:
        chosen = args.exchange if world > 1 else "single"
    graph = prepare(chosen)
    # ---- timed region: K steps, per-step events, L2 flush between steps
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    kev = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in jobs]
           for _ in range(args.steps)]
    sampler = ClockSampler(local)
    barrier()
    host_ms = []
    with sampler:
        for k in range(args.steps):
            flush.zero_()
            ev[k][0].record(stream)
            t_host = time.perf_counter()
            if graph is not None:
                graph.replay()
            else:
                step(kev[k])
            host_ms.append((time.perf_counter() - t_host) * 1e3)  # CPU time to enqueue the step's work
            ev[k][1].record(stream)
        barrier()
    host_enqueue_ms = float(np.median(host_ms))
    if mode == "sync":
        for j in jobs:
            j["dp"].check()
    step_ms = np.array([a.elapsed_time(b) for a, b in ev])
    if graph is not None:  # the graph step is timed whole: attribute it to the configs by pair count
        share = np.array([j["info"]["pairs"] for j in jobs], dtype=np.float64)
        kern_ms = step_ms[:, None] * (share / share.sum())[None, :]
    else:
        kern_ms = np.array([[a.elapsed_time(b) for a, b in row] for row in kev])  # [K, jobs]
    total_ms = max_over_ranks(float(step_ms.sum()))
    ms_per_step = total_ms / args.steps
    value = pairs_step / (ms_per_step * 1e-3)

    # ---- roofline of the dominant kernel (the P2P kernel).  Per config the floor is
    # max(pairs / MUFU peak, algorithmic bytes / HBM peak); the workload is
    # "alu"-bound (MUFU.LG2) when the MUFU floors dominate the sum, else "hbm"-bound.
    clocks = sampler.summary()
    peak_clk = (clocks["sm_max_mhz"] or 1965) * 1e6
    peak_mufu = MUFU_LG2_PER_CLK_PER_SM * SM_COUNT * peak_clk / 1e9  # Gpair/s
    peak_hbm, hbm_basis = _hbm_peak()
    kernel_ms = float(kern_ms.sum(axis=0).sum() / args.steps)
    alg_bytes = sum(j["info"]["alg_bytes_kernel"] for j in jobs)
    t_mufu = sum(j["info"]["pairs"] / (peak_mufu * 1e9) for j in jobs)
    t_hbm = sum(j["info"]["alg_bytes_kernel"] / (peak_hbm * 1e9) for j in jobs)
    traffic = _ncu_traffic(args, [j["name"] for j in jobs]) if world == 1 else None
    if args.kernel in MUFU_PER_PAIR_3D:  # 3D: MUFU ops per pair (RSQ [+ SIN + COS])
        m = MUFU_PER_PAIR_3D[args.kernel]
        achieved = pairs_local / (kernel_ms * 1e-3) / 1e9
        roofline = {"bound": "alu", "achieved": achieved, "peak": peak_mufu / m,
                    "unit": f"Gpair/s ({m} MUFU per pair)", "frac": achieved / (peak_mufu / m), "traffic": traffic,
                    "peak_basis": f"{MUFU_LG2_PER_CLK_PER_SM:.2f} MUFU/clk/SM x {SM_COUNT} SMs x {peak_clk / 1e6:.0f} MHz "
                                  f"/ {m} per pair; DESIGN.md §9e"}
    elif args.kernel == "helmholtz":  # FMA-pipe bound at the algorithm's op count
        achieved = pairs_local / (kernel_ms * 1e-3) / 1e9
        ops = HELM_OPS_PER_PAIR[args.precision]
        per_clk = FFMA_PER_CLK_PER_SM if args.precision == "fp32" else DFMA_PER_CLK_PER_SM
        peak = per_clk * SM_COUNT * peak_clk / ops / 1e9
        roofline = {"bound": "alu", "achieved": achieved, "peak": peak,
                    "unit": f"Gpair/s ({ops} {'FP32' if args.precision == 'fp32' else 'FP64'} FMA-pipe ops per pair)",
                    "frac": achieved / peak, "traffic": traffic,
                    "peak_basis": f"{per_clk:.1f} FMA/clk/SM x {SM_COUNT} SMs x {peak_clk / 1e6:.0f} MHz / {ops} ops "
                                  f"per pair (the series branch's algorithmic count, DESIGN.md §9c); {PEAK_BASIS}"}
    elif t_mufu >= t_hbm:
        achieved = pairs_local / (kernel_ms * 1e-3) / 1e9
        roofline = {"bound": "alu", "achieved": achieved, "peak": peak_mufu, "unit": "Gpair/s (1 MUFU.LG2 per pair)",
                    "frac": achieved / peak_mufu, "traffic": traffic,
                    "peak_basis": f"{MUFU_LG2_PER_CLK_PER_SM:.2f} MUFU.LG2/clk/SM x {SM_COUNT} SMs x "
                                  f"{peak_clk / 1e6:.0f} MHz (sm_max); {PEAK_BASIS}"}
    else:
        achieved = alg_bytes / (kernel_ms * 1e-3) / 1e9
        roofline = {"bound": "hbm", "achieved": achieved, "peak": peak_hbm, "unit": "GB/s (algorithmic bytes)",
                    "frac": achieved / peak_hbm, "traffic": traffic, "peak_basis": hbm_basis}
    roofline.update({"kernel_ms_per_step": kernel_ms, "alg_bytes_per_step": alg_bytes,
                     "hbm_gbs_alg": alg_bytes / (kernel_ms * 1e-3) / 1e9,
                     "mufu_frac": pairs_local / (kernel_ms * 1e-3) / 1e9 / peak_mufu,
                     "floor_frac": max(t_mufu, t_hbm) / (kernel_ms * 1e-3)})
    # the same bytes without SURVEY §8(d)'s 8 B per box of CSR offsets (the TILED kernel reads its
    # region tables instead): points only, 12 B per target + 12 B per source (fp32)
    pts_bytes = sum(3 * (4 if args.precision == "fp32" else 8) * (j["info"]["n_tgt_local"] + j["info"]["n_src_local"])
                    for j in jobs)
    roofline.update({"alg_bytes_points_only": pts_bytes,
                     "hbm_frac_points_only": pts_bytes / (kernel_ms * 1e-3) / 1e9 / peak_hbm})
    per_cfg = []
    for i, j in enumerate(jobs):
        kms = float(np.mean(kern_ms[:, i]))
        gp = j["info"]["pairs"] / (kms * 1e-3) / 1e9
        ab = j["info"]["alg_bytes_kernel"] / (kms * 1e-3) / 1e9
        per_cfg.append({"config": j["name"], "pairs": j["info"]["pairs"], "ms": kms, "Gpair_s": gp,
                        "frac_mufu": gp / peak_mufu, "alg_GBs": ab, "frac_hbm": ab / peak_hbm,
                        "layout_GBs": j["info"]["layout_bytes_apply"] / (kms * 1e-3) / 1e9,
                        "tile_log2": j["info"]["tile_log2"], "D_occ": j["info"]["density_occupied"],
                        "t_max": j["info"]["t_max"]})

    # ---- e2e through the C ABI with host buffers (pinned), copies inside the timed region
    args.exchange_chosen = mode
    e2e = None if args.no_e2e else _e2e(args, jobs, world, rank, stream, dev, pairs_step, barrier)

    out = {
        "metric": METRIC, "value": value, "unit": "pair-interactions/s", "n_gpus": world, "steps": args.steps,
        "warmup": max(3, args.warmup), "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "f32" if args.precision == "fp32" else "f64",
        "data": "synthetic (seeded SplitMix64 plates shaped like the paper's PEC plate, SURVEY.md §8(d))",
        "config": {"workload": args.workload + (f" x{world} (plates widened, weak scaling)" if weak else ""),
                   "configs": [j["cfg"].name for j in jobs], "layout": args.layout,
                   "precision": args.precision, "kind": args.kind, "pairs_per_step": pairs_step,
                   "kernel": args.kernel, **({"kappa_h": args.kh} if args.kernel.startswith("helmholtz") else {}),
                   "order": "plan", "l2": "flushed (256 MiB write) between timed steps",
                   "parallelism": f"morton-range x{world}" + (_exchange_desc(mode, shared, graph is not None)
                                                              if world > 1 else ""),
                   **({"exchange": mode, "exchange_autotune_ms": autotune} if world > 1 else {})},
        "gpu_launches": args.steps * len(jobs) * {"single": 1, "sync": 4, "nccl": 3, "peer": 2}[mode],
        # host-side cost of issuing one step's apply work (median over steps, max over ranks) against
        # the device step time: an enqueue shorter than the GPU step is not host-bound (N > 1 sync:
        # one graph launch); the L2-flush memset outside it can block on queue backpressure
        "host_enqueue_ms_per_step": max_over_ranks(host_enqueue_ms),
        "roofline": roofline, "clocks": clocks, "e2e": e2e, "per_config": per_cfg,
    }
    if world == 1 and args.precision == "fp32" and args.kernel == "laplace" and not args.profile:
        out["fp64"] = _fp64_line(args, names, stream, dev, flush, peak_clk)
    if rank == 0 and world == 1 and not args.no_cpu_baseline and not args.profile:
        out["cpu_baseline"] = {k: v for k, v in cpu_baseline(names, args.kind, args.cpu_seconds, kernel=args.kernel,
                                                             kh=args.kh).items()
                               if k not in ("pairs", "seconds")}
    if rank == 0 and world == 1 and not args.profile and args.layout in ("nr", "tiled") and not args.kernel.endswith("3d"):
        out["plan_build"] = _plan_build(args, jobs, dev)
    if rank == 0 and world == 1 and not args.no_extras and not args.profile:
        out["extras"] = _extras(args, names, stream, dev)
    for j in jobs:
        j["plan"].close()
    if rank == 0:
        print(json.dumps(out))
    if world > 1:
        dist.destroy_process_group()
    return 0


def _fp64_line(args, names, stream, dev, flush, peak_clk):
    """The same step in fp64 (the paper's precision): plans built the same way,
    K timed steps with the L2 flushed between them; roofline against the FP64 pipe at
    FP64_DP_OPS_PER_PAIR DP operations per pair and the measured DFMA rate."""
    import torch
    from paper_2403_01596_b200 import p2p
    plans, qs, outs, pairs = [], [], [], 0
    for name in names:
        cfg = W.CONFIGS[name]
        src, tgt, q = W.make_problem(cfg, kind=args.kind)
        kw = dict(level=cfg.level, layout=args.layout, precision="fp64", tile_log2=args.tile)
        if args.build == "device" and args.layout in ("nr", "tiled"):
            pl = p2p.Plan(torch.as_tensor(src, device=dev), torch.as_tensor(tgt, device=dev), device=dev.index,
                          build="device", **kw)
        else:
            pl = p2p.Plan(src, tgt, device=dev.index, **kw)
        plans.append(pl)
        qs.append(torch.as_tensor(q[pl.export("src_perm")], dtype=torch.float64, device=dev))
        outs.append(torch.empty(max(1, pl.info["n_tgt_local"]), dtype=torch.float64, device=dev))
        pairs += pl.info["pairs"]

    def step():
        for pl, q, o in zip(plans, qs, outs):
            p2p.p2p_apply(pl.handle, q.data_ptr(), o.data_ptr(), p2p.P2P_ORDER_PLAN, 0, stream.cuda_stream)

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize(dev)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for a, b in ev:
        flush.zero_()
        a.record(stream)
        step()
        b.record(stream)
    torch.cuda.synchronize(dev)
    ms = float(np.mean([a.elapsed_time(b) for a, b in ev]))
    for pl in plans:
        pl.close()
    achieved = pairs / (ms * 1e-3) / 1e9
    peak = DFMA_PER_CLK_PER_SM * SM_COUNT * peak_clk / FP64_DP_OPS_PER_PAIR / 1e9
    return {"value": pairs / (ms * 1e-3), "unit": "pair-interactions/s", "ms_per_step": ms, "dtype": "f64",
            "roofline": {"bound": "alu", "achieved": achieved, "peak": peak, "frac": achieved / peak,
                         "unit": f"Gpair/s ({FP64_DP_OPS_PER_PAIR} DP ops per pair on the FP64 pipe)",
                         "peak_basis": f"{DFMA_PER_CLK_PER_SM:.2f} DFMA/clk/SM x {SM_COUNT} SMs x "
                                       f"{peak_clk / 1e6:.0f} MHz / {FP64_DP_OPS_PER_PAIR}; {PEAK_BASIS}"}}


def _exchange_desc(mode, shared, graph):
    d = {"sync": " + halo pulled from the owners' HBM by one-sided peer reads ordered by device-side signal "
                 "words (p2p_apply_peer_sync; CUDA IPC / NVLink)" + (", step captured in a CUDA graph" if graph else ""),
         "nccl": " + NCCL halo exchange (torch.distributed all_to_all)",
         "peer": " + peer-memory halo (CUDA IPC / NVLink) with host barriers"}[mode]
    if shared:
        d += ("" if mode != "nccl" else " staged through the host over gloo") + ", ranks sharing GPUs (TEST MODE)"
    return d


def _e2e_dist(args, jobs, stream, pairs_step, barrier):
    """N > 1: each rank's public-API step from host memory: H2D of its owned weights (pinned),
    halo exchange + distributed apply (DistributedP2P.apply), D2H of its potentials; time = max
    over ranks."""
    import torch
    import torch.distributed as dist
    hq = [j["q_owned"].cpu().pin_memory() for j in jobs]
    ho = [torch.empty_like(j["out"], device="cpu").pin_memory() for j in jobs]
    dq = [torch.empty_like(j["q_owned"]) for j in jobs]
    h2d = sum(int(t.numel() * t.element_size()) for t in hq)
    d2h = sum(int(t.numel() * t.element_size()) for t in ho)

    comm = torch.cuda.Stream()
    sync = getattr(args, "exchange_chosen", args.exchange) == "sync"

    def step():
        for a, d in zip(hq, dq):
            d.copy_(a, non_blocking=True)
        if sync:  # device-synchronised peer exchange: stream-ordered, no host work between ranks
            for j, d, b in zip(jobs, dq, ho):
                j["dp"].apply_sync(d, j["out"], stream=stream.cuda_stream)
                b.copy_(j["out"], non_blocking=True)
            return
        comm.wait_stream(torch.cuda.current_stream())
        ready = [j["dp"].exchange_async(d, comm) for j, d in zip(jobs, dq)]
        for j, d, b, ev in zip(jobs, dq, ho, ready):
            j["dp"].apply(d, j["out"], stream=stream.cuda_stream, halo_ready=ev)
            b.copy_(j["out"], non_blocking=True)

    for _ in range(3):
        step()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    barrier()
    t = torch.tensor([e0.elapsed_time(e1) / args.steps], dtype=torch.float64)
    if dist.get_backend() == "nccl":
        t = t.cuda()
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    return {"value": pairs_step / (ms * 1e-3), "unit": "pair-interactions/s", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "ms_per_step": ms,
            "path": "per rank: pinned H2D of owned weights, " + (
                "p2p_apply_peer_sync (halo pulled from the owners' memory, device-side signals)" if sync else
                "halo exchanges (DistributedP2P.exchange_async on a comm stream) overlapping the previous "
                "config's p2p_apply_dist") + ", D2H of local potentials; max over ranks"}


def src_sha16():
    """Hash of the operator's sources (csrc/ + include/): ties a committed ncu summary to the code
    it was captured on."""
    import hashlib
    h = hashlib.sha256()
    for d in (os.path.join(ROOT, "paper_2403_01596_b200", "csrc"), os.path.join(ROOT, "include")):
        for f in sorted(os.listdir(d)):
            if f.endswith((".cu", ".cuh", ".cpp", ".h")):
                h.update(f.encode())
                h.update(open(os.path.join(d, f), "rb").read())
    return h.hexdigest()[:16]


def _ncu_traffic(args, names):
    """dram bytes per launch of the P2P kernel from the committed ncu --set full summary
    (profiles/ncu_summary.json, tools/ncu_traffic_json.py), only if it was captured on these
    sources (same src_sha16); else None."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        data = json.load(open(path))
        key = f"{args.layout}_{args.precision}"
        sha = src_sha16()
        ents = [data[n][key] for n in names if n in data and key in data[n]]
        if len(ents) != len(names) or any(e.get("src_sha16") != sha for e in ents):
            return None
        return float(sum(e["dram_bytes"] for e in ents))
    except Exception:
        return None


def _e2e(args, jobs, world, rank, stream, dev, pairs_step, barrier):
    """Same metric through the C ABI with pinned HOST buffers (p2p_apply_host_async): every
    step copies q host->device, applies (user order: permutation kernels included), copies phi
    device->host.  Steps are pipelined the way a serving loop runs them: each plan has three
    workspace slots (p2p_plan_set_workspaces) and consecutive steps rotate over three streams
    per config, so step k's D2H overlaps step k+1's H2D and kernel (each apply waits on
    the device for the apply that last used its slot)."""
    import torch
    from paper_2403_01596_b200 import p2p
    if world > 1:
        return _e2e_dist(args, jobs, stream, pairs_step, barrier)
    hq = [torch.as_tensor(j["q_user"], dtype=j["plan"].torch_dtype).pin_memory() for j in jobs]
    NS = 3
    ho = [[torch.empty(j["info"]["n_tgt"], dtype=j["plan"].torch_dtype).pin_memory() for _ in range(NS)]
          for j in jobs]
    h2d = sum(int(t.numel() * t.element_size()) for t in hq)
    d2h = sum(int(t[0].numel() * t[0].element_size()) for t in ho)
    for j in jobs:
        j["plan"].set_workspaces(NS)
    side = [[torch.cuda.Stream(dev) for _ in range(NS)] for _ in jobs]

    def run(steps):
        start = torch.cuda.Event()
        start.record(stream)
        for ss in side:
            for st in ss:
                st.wait_event(start)
        for k in range(steps):
            for j, a, b, ss in zip(jobs, hq, ho, side):
                st = ss[k % NS]
                p2p.p2p_apply_host_async(j["plan"].handle, a.data_ptr(), b[k % NS].data_ptr(), p2p.P2P_ORDER_USER, 0,
                                         st.cuda_stream)
        for ss in side:
            for st in ss:
                done = torch.cuda.Event()
                done.record(st)
                stream.wait_event(done)

    run(3)
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    run(args.steps)
    e1.record(stream)
    barrier()
    ms = e0.elapsed_time(e1) / args.steps
    return {"value": pairs_step / (ms * 1e-3), "unit": "pair-interactions/s", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "ms_per_step": ms,
            "path": "p2p_apply_host_async, pinned host buffers, user order; three workspace slots per plan, "
                    "consecutive steps on rotating streams (step k's D2H overlaps step k+1's H2D + kernel)"}


def _plan_build(args, jobs, dev):
    """The paper's "collection" (plan build) of the step's configs: host C++ builder (+ upload)
    vs the device builder (p2p_plan_create_device, coordinates already in HBM); same plan."""
    import torch
    from paper_2403_01596_b200 import p2p
    host = dev_s = 0.0
    for j in jobs:
        cfg = j["cfg"]
        src, tgt, _ = W.make_problem(cfg, kind=args.kind)
        kw = dict(level=cfg.level, layout=args.layout, precision=args.precision, tile_log2=args.tile,
                  **_kernel_kw(args, cfg))
        with p2p.Plan(src, tgt, device=dev.index, **kw) as pl:
            host += pl.info["build_seconds"] + pl.info["upload_seconds"]
        ds, dt = torch.as_tensor(src, device=dev), torch.as_tensor(tgt, device=dev)
        best = float("inf")
        for _ in range(2):
            with p2p.Plan(ds, dt, device=dev.index, build="device", **kw) as pl:
                best = min(best, pl.info["build_seconds"])
        dev_s += best
    return {"host_build_upload_s": host, "device_build_s": dev_s, "speedup": host / dev_s,
            "host_cores": len(os.sched_getaffinity(0)), "step_plans": args.build,
            "note": "same plan either way (tests/test_device_plan.py: every export and apply bit-identical)"}


def _extras(args, names, stream, dev):
    """Detail lines: both layouts x both precisions on the same workload (fewer steps)."""
    import torch
    from paper_2403_01596_b200 import p2p
    res = []
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    for layout in ("nr", "r", "tiled"):
        for prec in ("fp32", "fp64"):
            for name in names:
                cfg = W.CONFIGS[name]
                src, tgt, q = W.make_problem(cfg, kind=args.kind)
                with p2p.Plan(src, tgt, level=cfg.level, layout=layout, precision=prec, device=dev.index) as pl:
                    qd = torch.as_tensor(q[pl.export("src_perm")], dtype=pl.torch_dtype, device=dev)
                    out = torch.empty(pl.info["n_tgt_local"], dtype=pl.torch_dtype, device=dev)
                    for _ in range(3):
                        pl.apply(qd, out)
                    times = []
                    for _ in range(5):
                        flush.zero_()
                        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                        a.record(stream)
                        pl.apply(qd, out)
                        b.record(stream)
                        b.synchronize()
                        times.append(a.elapsed_time(b))
                    ms = float(np.median(times))
                    info = pl.info
                    res.append({"config": name, "layout": layout, "precision": prec, "ms": ms,
                                "Gpair_s": info["pairs"] / (ms * 1e-3) / 1e9,
                                "alg_GBs": info["alg_bytes_kernel"] / (ms * 1e-3) / 1e9,
                                "layout_GBs": info["layout_bytes_apply"] / (ms * 1e-3) / 1e9,
                                "plan_build_s": info["build_seconds"], "upload_s": info["upload_seconds"],
                                "device_MB": info["device_bytes"] / 1e6, "halo_entries": info["halo_entries"]})
    return res


if __name__ == "__main__":
    sys.exit(main())
