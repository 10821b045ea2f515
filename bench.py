#!/usr/bin/env python
"""KITC hot-path benchmark (driver contract).

Step = one pass of the whole hot path over one synthetic input: tree build +
modified weights (this rank's cluster shard) [+ NCCL all-gather of fhat] +
treecode evaluation of this rank's targets, for BASELINE.json config C3
(N = 1e6 uniform, Stokeslet, n = 8, theta = 0.7, N0 = 2000, eps = 0.01).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3]
  python bench.py --impl reference ...   # the CPU oracle, bounded sample

Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import kitc_inputs as KI  # noqa: E402

METRIC = "KITC Stokeslet targets/s, N=1e6 n=8 θ=0.7, 1/2/4/8 B200; % of FP64 peak"
KNAME = {0: "Stokeslet", 1: "rotlet", 2: "Stokeslet+rotlet"}


def metric_for(config):
    """BASELINE.json's metric for the headline config C3; the same wording for the others."""
    if config == "C3":
        return METRIC
    c = KI.CONFIGS[config]
    return f"KITC {KNAME[c['kernel']]} targets/s, N={c['N']:.0e} n={c['n']} θ={c['theta']} ({config}); % of FP64 peak"
UNIT = "targets/s"
FLOPS_PER_PAIR = {0: 32, 1: 59, 2: 91}   # algorithmic flops per pair
PEAK_SMS, PEAK_FMA_PER_CLK = 148, 64     # B200: 148 SMs x 64 FP64 FMA/clk/SM


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="kitc", choices=["kitc", "reference"])
    ap.add_argument("--config", default="C3")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-check", action="store_true", help="skip E vs the GPU direct sum")
    ap.add_argument("--exchange", default="p2p", choices=["p2p", "nccl"],
                    help="N>1 fhat exchange: fused peer-memory stores (default) or NCCL all-gather")
    ap.add_argument("--dry-run", action="store_true",
                    help="launcher check: start the ranks, one all-reduce (gloo without a GPU), print the rank count")
    return ap.parse_args()


def workload(config):
    """The `config.workload` string -- identical in both arms."""
    return f"{config} ({KI.CONFIGS[config]})"


PRECISION = ("fp64 throughout; the treecode evaluation's s^-1/2 is one Newton step from the MUFU seed "
             "(relative error < 2e-12, DESIGN.md reading A19); the direct sum keeps ~4 ulp")


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi sampling during the timed region (recipe's clocks line)."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.p = None
        self.path = os.path.join("/tmp", f"kitc_clocks_{os.getpid()}.csv")

    def start(self):
        """Start nvidia-smi and wait (<= 5 s) until it has produced its first line, so that the
        samples taken from `mark()` on cover the timed region even when it is short."""
        try:
            self.f = open(self.path, "w")
            self.p = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "20"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
            t0 = time.time()
            while time.time() - t0 < 5.0 and os.path.getsize(self.path) == 0:
                time.sleep(0.01)
        except Exception:
            self.p = None
        self.pos = 0

    def mark(self):
        """The timed region starts: later lines only."""
        try:
            self.f.flush()
            self.pos = os.path.getsize(self.path)
        except Exception:
            self.pos = 0

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        self.f.close()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        with open(self.path) as fh:
            fh.seek(self.pos)
            lines = fh.read().splitlines()
        for line in lines:
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax.append(float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        os.unlink(self.path)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------- oracle leg
_ORC = {}  # state shared with forked oracle workers (copy-on-write)


def _orc_weights(rng):
    t0 = time.perf_counter()
    _ORC["T"].modified_weights(_ORC["W"], _ORC["n"], cluster_range=rng, out=_ORC["F"].copy())
    return time.perf_counter() - t0


def _orc_eval(tg):
    c = _ORC["cfg"]
    t0 = time.perf_counter()
    _ORC["T"].treecode(c["kernel"], c["eps"], c["n"], c["theta"], _ORC["W"], fhat=_ORC["F"], targets=tg)
    return time.perf_counter() - t0


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def oracle_sample(cfg, X, W, S_targets, weight_frac=0.1, seed=1, fhat=None, procs=1):
    """Bounded sample of the CPU oracle on the workload: full tree build,
    Algorithm 1 on a set of clusters holding >= weight_frac of sum N_C
    (extrapolated by sum N_C), Algorithm 2 on S_targets random targets
    (extrapolated by N / S).  procs > 1: the weights clusters and the sampled
    targets are split over `procs` forked processes running the same
    single-threaded oracle (the whole host), time = the slowest process; the
    tree build stays one process.  Returns (targets/s, detail, fhat)."""
    import oracle as O
    N = cfg["N"]
    t0 = time.perf_counter()
    T = O.Tree(X, cfg["N0"])
    t_tree = time.perf_counter() - t0
    sizes = T.end - T.begin
    tot = float(sizes[1:].sum())        # root skipped on both sides (reading A16)
    cb = T.nclusters
    acc = 0.0
    while cb > 1 and acc < weight_frac * tot:
        cb -= 1
        acc += sizes[cb]
    m = O.DIMS[cfg["kernel"]][0]
    F = np.zeros((T.nclusters, m, (cfg["n"] + 1) ** 3)) if fhat is None else fhat.copy()
    tg = KI.sample_targets(N, S_targets, seed=seed)
    w_scale = tot / acc if acc > 0 else 0.0
    e_scale = N / len(tg)
    if procs <= 1:
        t0 = time.perf_counter()
        T.modified_weights(W, cfg["n"], cluster_range=(cb, T.nclusters), out=F)
        t_w_raw = time.perf_counter() - t0
        if fhat is None:
            F = T.modified_weights(W, cfg["n"], cluster_range=(1, T.nclusters), out=F)
        t0 = time.perf_counter()
        T.treecode(cfg["kernel"], cfg["eps"], cfg["n"], cfg["theta"], W, fhat=F, targets=tg)
        t_e_raw = time.perf_counter() - t0
    else:
        import multiprocessing as mp
        if fhat is None:
            F = T.modified_weights(W, cfg["n"], cluster_range=(1, T.nclusters), out=F)
        _ORC.update(T=T, W=W, F=F, n=cfg["n"], cfg=cfg)
        cum = np.concatenate([[0.0], np.cumsum(sizes[cb:].astype(np.float64))])
        cuts = [cb + int(np.searchsorted(cum, cum[-1] * r / procs)) for r in range(procs)] + [T.nclusters]
        wr = [(b, e) for b, e in zip(cuts[:-1], cuts[1:]) if e > b]   # cluster ranges balanced by N_C
        with mp.get_context("fork").Pool(procs) as pool:
            t_w_raw = max(pool.map(_orc_weights, wr)) if (acc > 0 and wr) else 0.0
            t_e_raw = max(pool.map(_orc_eval, np.array_split(tg, procs)))
        _ORC.clear()
    t_w, t_e = t_w_raw * w_scale, t_e_raw * e_scale
    total = t_tree + t_w + t_e
    return N / total, dict(t_tree_s=t_tree, t_weights_sample_s=t_w_raw, weights_scale=w_scale,
                           t_weights_s_extrapolated=t_w, t_eval_sample_s=t_e_raw, eval_scale=e_scale,
                           t_eval_s_extrapolated=t_e, sample_wall_s=t_tree + t_w_raw + t_e_raw,
                           weight_clusters=int(T.nclusters - cb), eval_targets=int(len(tg)),
                           processes=procs), F


def run_reference(args, cfg, rank, world):
    if rank != 0:
        return
    X, W = KI.config_particles(args.config)
    import oracle as O
    O.build()
    # untimed setup: full modified weights so the sampled evaluation reads real data
    _, _, F = oracle_sample(cfg, X, W, 50, weight_frac=0.0)
    procs = host_cores()
    S = 100 * procs
    times, dets = [], []
    for i in range(args.warmup + args.steps):
        v, det, _ = oracle_sample(cfg, X, W, S, seed=100 + i, fhat=F, procs=procs)
        if i >= args.warmup:
            times.append(cfg["N"] / v)
            dets.append(det)
    tstep = sum(times) / len(times)
    val = cfg["N"] / tstep
    measured = {k: sum(d[k] for d in dets) / len(dets) for k in
                ("t_tree_s", "t_weights_sample_s", "weights_scale", "t_eval_sample_s", "eval_scale", "sample_wall_s")}
    sample = (f"per step: full oracle tree build (1 process); Algorithm 1 on the last clusters holding >=10% of "
              f"sum N_C (time x sum N_C ratio) and Algorithm 2 on {S} random targets (time x N/{S}), both split "
              f"over {procs} processes of the single-threaded oracle (slowest process timed)")
    line = {"impl": "reference", "metric": metric_for(args.config), "value": val, "unit": UNIT,
            "n_gpus": max(world, args.gpus), "steps": args.steps, "warmup": args.warmup, "ms_per_step": tstep * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "precision": "fp64, long double per-target accumulators (the CPU oracle, oracle/kitc_oracle.c)",
            "data": data_str(cfg), "config": {"workload": workload(args.config)},
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": procs, "kind": "oracle", "sample": sample,
                             "measured_per_step": measured,
                             "note": "time per step = t_tree + t_weights_sample x weights_scale + "
                                     "t_eval_sample x eval_scale (extrapolated; sample_wall_s is what ran)"},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def data_str(cfg):
    return "synthetic (kitc_inputs: " + (
        "organism pairs of the paper's Example 1, unit forces +-t" if cfg["geometry"] == "organisms"
        else f"{cfg['geometry']}, weights uniform [-1,1]^m") + ", seed 0)"


def probe_fp64_peak(seconds=0.5):
    """DFMA rate measured on this box (tools/libfp64_peak.so, untimed, before the timed region)."""
    import ctypes as Cc
    try:
        L = Cc.CDLL(os.path.join(ROOT, "tools", "libfp64_peak.so"))
        L.kitc_probe_dfma_tflops.argtypes = [Cc.c_double, Cc.POINTER(Cc.c_double), Cc.POINTER(Cc.c_double)]
        tf, fc = Cc.c_double(), Cc.c_double()
        if L.kitc_probe_dfma_tflops(seconds, Cc.byref(tf), Cc.byref(fc)) != 0:
            return None
        return {"tflops": tf.value, "fma_per_sm_clk_at_max_clock": fc.value,
                "how": f"tools/fp64_peak.cu: 148 SMs x 4 CTAs x 256 threads, 8 independent DFMA chains, {seconds} s"}
    except OSError:
        return None


# ----------------------------------------------------------------------------- GPU leg
def run_kitc(args, cfg, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    from paper_1902_02250_b200 import dist as D
    from paper_1902_02250_b200 import kitc

    kern, n, theta, N0, eps, N = cfg["kernel"], cfg["n"], cfg["theta"], cfg["N0"], cfg["eps"], cfg["N"]
    X, W = KI.config_particles(args.config)
    # oracle baseline first: it forks worker processes, which must happen before CUDA is initialised
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        import oracle as O
        O.build()
        procs = host_cores()
        v1, det1, F1 = oracle_sample(cfg, X, W, 1500)
        v, det, _ = oracle_sample(cfg, X, W, 200 * procs, seed=2, fhat=F1, procs=procs)
        del F1
        cpu = {"value": v, "unit": UNIT, "cores": procs, "kind": "oracle",
               "sample": f"full oracle tree (1 process); Algorithm 1 on clusters holding >=10% of sum N_C "
                         f"(x sum N_C ratio) and Algorithm 2 on {200 * procs} random targets (x N/{200 * procs}), "
                         f"split over {procs} processes of the single-threaded oracle (slowest timed)", **det,
               "single_core": {"value": v1, "cores": 1, "eval_targets": 1500, **det1}}

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    stream = torch.cuda.current_stream()
    m, p = kitc.kitc_kernel_dims(kern)
    P3 = (n + 1) ** 3
    Xd = torch.from_numpy(X).to(dev)
    Wd = torch.from_numpy(W).to(dev)
    T = kitc.Tree(Xd, N0)
    C = T.nclusters
    rg = T.export_ranges()
    if world > 1:  # every rank must have built the identical tree (deterministic build): compare a checksum
        h = torch.tensor([float(np.sum((rg["begin"] * 1000003 + rg["end"]) % 998244353)), float(C)],
                         dtype=torch.float64, device=dev)
        lo, hi = h.clone(), h.clone()
        dist.all_reduce(lo, op=dist.ReduceOp.MIN)
        dist.all_reduce(hi, op=dist.ReduceOp.MAX)
        if not torch.equal(lo, hi):
            raise RuntimeError("ranks built different trees")
    cshards = D.cluster_shards(rg["begin"], rg["end"], world, skip_root=True)   # targets = sources, theta < 1 (A16)
    S = D.padded_shard_size(cshards)
    cb, ce = cshards[rank]
    L = kitc.kitc_fhat_cluster_len(kern, n)
    gathered = torch.zeros((world, S, L), dtype=torch.float64, device=dev)
    fhat = torch.zeros((C, L), dtype=torch.float64, device=dev)
    out = torch.zeros((N, p), dtype=torch.float64, device=dev)
    row = L * 8
    shard_base = gathered[rank].data_ptr() - cb * row    # virtual base: cluster c -> shard row c - cb
    import ctypes as Cc

    def weights_nccl():
        kitc.kitc_modified_weights(T.handle, kern, n, kitc._ptr(Wd), cb, ce, Cc.c_void_p(shard_base),
                                   kitc._stream())
        D.all_gather_fhat(fhat, gathered, gathered[rank], cshards, rank)

    exchange = "none (1 GPU)" if world == 1 else "NCCL all_gather_into_tensor of padded fhat shards"
    use_p2p = world > 1 and args.exchange == "p2p"
    if use_p2p:
        # fused weights + exchange over peer memory; cross-checked bitwise against the NCCL path
        why = ""
        try:
            pf = D.PeerFhat(C, L, dev)
            fhat_p2p = pf.modified_weights(T, kern, n, Wd, (cb, ce))
            torch.cuda.synchronize()
        except Exception as ex:  # symmetric memory unavailable on this node: say so, use NCCL
            why = f"{type(ex).__name__}: {ex}"
        okf = torch.tensor([0 if why else 1], device=dev)
        dist.all_reduce(okf, op=dist.ReduceOp.MIN)   # one decision for all ranks
        if int(okf[0]) != 1:
            use_p2p = False
            exchange = f"NCCL all_gather_into_tensor (peer-memory path unavailable: {why or 'on another rank'})"[:300]
    if use_p2p:
        weights_nccl()
        torch.cuda.synchronize()
        ok = torch.tensor([int(torch.equal(fhat_p2p[1:], fhat[1:]))], device=dev)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        if int(ok[0]) != 1:
            raise RuntimeError("fused peer-memory fhat differs from the NCCL all-gather")
        fhat = fhat_p2p
        exchange = f"fused modified weights -> {world} peer replicas (symmetric memory, device barriers)"

    def weights():
        if world == 1:
            T.modified_weights(kern, n, Wd, cluster_range=(cb, ce), fhat=fhat)
        elif use_p2p:
            pf.modified_weights(T, kern, n, Wd, (cb, ce))
        else:
            weights_nccl()

    ev_e0, ev_e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def step(Xsrc=None, timed_eval=False):
        T.build(Xd if Xsrc is None else Xsrc, N0)
        weights()
        if timed_eval:
            ev_e0.record(stream)
        T.eval(kern, n, theta, eps, fhat, out=out, part=(rank, world))
        if timed_eval:
            ev_e1.record(stream)

    # algorithmic work of this rank's eval launch (interaction counts, deterministic)
    step()
    _, st = T.eval(kern, n, theta, eps, fhat, part=(rank, world), stats=True)
    torch.cuda.synchronize()
    st = st.cpu().numpy()
    pairs = int(st[:, 1].sum() + st[:, 3].sum())
    flops_eval = pairs * FLOPS_PER_PAIR[kern]

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)   # 256 MB > 126 MB L2
    for _ in range(max(3, args.warmup)):
        step()
    barrier()
    clk = ClockSampler(local_rank)
    clk.start()
    clk.mark()
    l0 = kitc.kitc_launch_count()
    tot_ms, eval_ms = 0.0, 0.0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(args.steps):
        flush.zero_()                               # L2 flushed between timed steps (untimed)
        e0.record(stream)
        step(timed_eval=True)
        e1.record(stream)
        e1.synchronize()
        tot_ms += e0.elapsed_time(e1)
        eval_ms += ev_e0.elapsed_time(ev_e1)
    launches = kitc.kitc_launch_count() - l0
    barrier()
    clocks = clk.stop()
    t = torch.tensor([tot_ms, eval_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_step = float(t[0]) / args.steps
    value = N / (ms_step / 1e3)
    eval_launch_ms = eval_ms / args.steps

    # e2e: host buffers through the C ABI, H2D + step + D2H inside the timed region.  The weights'
    # upload runs on a second stream beside the tree build (it is needed only by the modified
    # weights), and the evaluation writes each target's row straight into the pinned host output
    # (mapped into the device address space: zero-copy, overlapped with the kernel) -- the same
    # bytes cross the host link every step, counted below.
    e2e = None
    if not args.no_e2e:
        Xh = torch.from_numpy(X).pin_memory()
        Wh = torch.from_numpy(W).pin_memory()
        outh = torch.empty((N, p), dtype=torch.float64).pin_memory()
        Xe = torch.empty_like(Xd)
        s2 = torch.cuda.Stream(device=dev)
        ev_w, ev_used = torch.cuda.Event(), torch.cuda.Event()
        ev_used.record(stream)

        def e2e_step():
            Xe.copy_(Xh, non_blocking=True)
            s2.wait_event(ev_used)                   # the previous step has gathered Wd
            with torch.cuda.stream(s2):
                Wd.copy_(Wh, non_blocking=True)
                ev_w.record(s2)
            T.build(Xe, N0)
            stream.wait_event(ev_w)
            weights()
            ev_used.record(stream)
            T.eval(kern, n, theta, eps, fhat, out=outh, part=(rank, world))

        e2e_step()
        barrier()
        tot = 0.0
        for _ in range(args.steps):
            flush.zero_()
            e0.record(stream)
            e2e_step()
            e1.record(stream)
            e1.synchronize()
            tot += e0.elapsed_time(e1)
        tt = torch.tensor([tot], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_ms = float(tt[0]) / args.steps
        torch.cuda.synchronize()
        same = bool(torch.equal(outh, out.cpu())) if world == 1 else None   # zero-copy output == device output
        e2e = {"value": N / (e2e_ms / 1e3), "unit": UNIT, "ms_per_step": e2e_ms,
               "h2d_bytes_per_step": int(X.nbytes + W.nbytes), "d2h_bytes_per_step": int(N * p * 8),
               "how": "pinned H2D of X (stream) and W (side stream, beside the tree build); the evaluation "
                      "writes the output rows into pinned host memory (zero-copy)",
               "host_output_equals_device_output": same}

    # accuracy of this run vs the GPU direct sum (outside every timed region)
    check = None
    if not args.no_check and world == 1:
        ref = kitc.direct(Xd, Wd, kern, eps)
        check = {"E_vs_gpu_direct": kitc.rel_error(ref, out)}

    probe = probe_fp64_peak() if rank == 0 else None
    if rank != 0:
        return
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    smax = float(peaks.get("sm_max_mhz", 1965.0))
    peak_tflops = PEAK_SMS * PEAK_FMA_PER_CLK * 2 * smax * 1e6 / 1e12
    achieved = flops_eval / (eval_launch_ms * 1e-3) / 1e12
    traffic, traffic_src = None, None
    from paper_1902_02250_b200 import build as B
    bid = B.build_id()
    traffic_build = None
    try:  # dram read + write bytes of one k_eval launch from the committed ncu --set full capture
        tr = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))[args.config]
        traffic, traffic_src, traffic_build = tr["dram_bytes_per_launch"], tr["source"], tr.get("build_id")
    except Exception:
        pass
    roof = {"bound": "alu", "kernel": "k_eval (treecode evaluation)", "achieved": achieved,
            "peak": peak_tflops, "unit": "TFLOP/s", "frac": achieved / peak_tflops, "traffic": traffic,
            "traffic_unit": "bytes per launch (ncu dram__bytes_read.sum + dram__bytes_write.sum)",
            "traffic_source": traffic_src, "build_id": bid, "traffic_build_id": traffic_build,
            "traffic_same_build": traffic_build == bid,
            "peak_source": f"derived (contract: ALU-bound peak from unit counts and clocks): {PEAK_SMS} SMs x "
                           f"{PEAK_FMA_PER_CLK} FP64 FMA/clk x 2 x {smax:.0f} MHz",
            "peak_measured": probe["tflops"] if probe else None,
            "frac_of_measured": (achieved / probe["tflops"]) if probe else None,
            "peak_measured_source": probe,
            "algorithmic_flops_per_launch": flops_eval, "pairs_per_launch": pairs,
            "flops_per_pair": FLOPS_PER_PAIR[kern], "launch_ms": eval_launch_ms,
            "step_share": eval_launch_ms / ms_step}
    line = {"metric": metric_for(args.config), "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "precision": PRECISION,
            "data": data_str(cfg),
            "config": {"workload": workload(args.config)},
            "setup": {"parallelism": f"tree replicated, fhat sharded, targets dp{world} (64-batch chunks interleaved)",
                      "fhat_exchange": exchange,
                      "l2": "flushed between timed steps (256 MB write, untimed)",
                      "clusters": C, "depth": T.depth, "batches": T.nbatches},
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "clocks": clocks, "check": check}
    print(json.dumps(line), flush=True)


def launch_ranks(args):
    """--gpus N > 1 without a torch.distributed environment: re-run this command under
    torch.distributed.run, one process per GPU (127.0.0.1 rendezvous)."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")           # communicator lines (rank count) on stderr
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd, env=env)


def dry_run(args, rank, world):
    import torch
    import torch.distributed as dist
    if world > 1:
        dist.init_process_group("nccl" if torch.cuda.is_available() else "gloo")
        t = torch.ones(1, device="cuda" if torch.cuda.is_available() else "cpu")
        dist.all_reduce(t)
        seen = int(t.item())
        dist.destroy_process_group()
    else:
        seen = 1
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "ranks_seen": seen, "gpus_arg": args.gpus}), flush=True)


def main():
    args = parse()
    cfg = dict(KI.CONFIGS[args.config])
    if "WORLD_SIZE" not in os.environ and args.gpus > 1 and args.impl != "reference":
        sys.exit(launch_ranks(args))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, cfg, rank, world)
        return
    if world != args.gpus:
        sys.exit(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}: one rank per GPU is required")
    if args.dry_run:
        dry_run(args, rank, world)
        return
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")   # communicator init lines show the rank count
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        import torch
        if torch.cuda.device_count() < world:
            sys.exit(f"bench.py: --gpus {world} but this node has {torch.cuda.device_count()} GPUs")
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_kitc(args, cfg, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
