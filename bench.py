#!/usr/bin/env python
"""FGA hot-path benchmark on B200 (contract: see DESIGN.md "Measurement").

Workload (BASELINE.json configs[2], the 1M-point FGA the metric is quoted
on): a 1,000,000 x 1,000,000 synthetic blob pair (synth.blob, PCG64 seed 3,
random rotation <= 60 deg, translation <= 0.1), Barnes-Hut theta = 0.5.  A
"step" is one FGA iteration: the force pass over the whole template
(traversal + fused Euler-Cromer step + Kabsch partials), the partial
reduction and the fp64 rigid update.  `value` = accepted particle-node
interactions per second (each accepted node is one softened pair
interaction, the reference's own unit: _kernels.py:37-42), whole job.

Extra legs in the same JSON line (N=1 only): `direct` (theta = 0, exact O(NM)
direct sum, pairs/s and its FP32 roofline), `e2e` (the reference-facing
bh_forces drop-in with pinned host buffers: H2D + traversal + D2H per step),
`registration` (full register() wall time from host arrays), `cpu_baseline`
(the C oracle on all host cores, bounded sample).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "particle-pair interactions/sec and registration wall-time, 1M-pt FGA, 1–8 B200"
UNIT = "interactions/s"
FLOP_PER_INTERACTION = 20  # GPU Gems 3 ch.31 n-body convention
FLOP_PER_VISIT = 9         # MAC: 3 sub + 5 (d^2) + 1 (theta^2 d^2)
BYTES_PER_VISIT = 32       # one 32 B node record per query-node visit
BYTES_PER_QUERY = 32       # + 16 B query in, 16 B state out per template point
BUILD_BYTES_PER_POINT = 350  # SURVEY §8(d) K2-K5 algorithmic bytes per reference point


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=1_000_000)
    ap.add_argument("--theta", type=float, default=0.5)
    ap.add_argument("--seed", type=int, default=3)
    ap.add_argument("--no-direct", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-registration", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--direct-steps", type=int, default=3)
    ap.add_argument("--no-batched", action="store_true")
    ap.add_argument("--no-build", action="store_true")
    ap.add_argument("--no-fp64", action="store_true")
    ap.add_argument("--no-ingest", action="store_true")
    ap.add_argument("--build-sizes", default="1000000,16000000")
    ap.add_argument("--no-configs", action="store_true",
                    help="skip the configs[1]/configs[3] registration legs")
    ap.add_argument("--batch-pairs", type=int, default=4096)
    ap.add_argument("--cpu-sample", type=int, default=65536)
    ap.add_argument("--default-g", action="store_true",
                    help="keep G=66.7 (diverges at 1M, SURVEY §0.11) instead of the "
                         "converging G*sqrt(2000/N)")
    return ap.parse_args()


def bench_params(args):
    """BASELINE configs[2] parameters: theta=0.5; G scaled by sqrt(2000/N) so
    the 1M registration converges (the reference's field
    mass grows as sqrt(N) while G stays fixed, which makes the default run
    fly apart above ~50k points).  The scaling is a user-level parameter
    applied identically to every arm."""
    import paper_2009_14005_b200 as fga
    p = fga.default_params().replace(theta=args.theta)
    if not args.default_g:
        p = p.replace(G=66.7 * (2000.0 / args.n) ** 0.5)
    return p


def workload(n, seed):
    from paper_2009_14005_b200 import synth
    return synth.configs2_pair(n, seed)


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0}, "fallback"


def fp32_peak_tflops(sm_mhz, sms=148):
    return 2.0 * sms * 128 * sm_mhz * 1e6 / 1e12


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = os.path.join("/tmp", f"fga_clocks_{os.getpid()}.csv")

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            time.sleep(0.15)
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        try:
            rows = [r.split(",") for r in open(self.path).read().strip().splitlines()]
        except OSError:
            rows = []
        rows = [[c.strip() for c in r] for r in rows if len(r) >= 7]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            for nm, v in zip(names, r[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": float(rows[0][1]) if rows[0][1].replace(".", "").isdigit() else None,
                "reasons": sorted(reasons), "samples": len(rows)}


# --------------------------------------------------------------------------- ours
def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    import paper_2009_14005_b200 as fga
    from paper_2009_14005_b200.engine import SUM_ACCEPTED, SUMS_LEN, Session

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    x, y = workload(args.n, args.seed)
    K, W = args.steps, args.warmup
    params = bench_params(args).replace(conv_tol=1e-300, max_iters=W + K + 1)
    opts = fga.RegisterOptions(compute_gpe=False)
    x_t = torch.from_numpy(np.array(x.points)).to(dev)
    y_t = torch.from_numpy(np.array(y.points)).to(dev)
    stream = torch.cuda.current_stream()
    sess = Session(None, None, params, opts, shard_rank=rank, shard_count=world,
                   device=local_rank, stream=stream.cuda_stream,
                   device_inputs=(x_t.data_ptr(), len(x), y_t.data_ptr(), len(y)))
    sums = torch.zeros(SUMS_LEN, dtype=torch.float64, device=dev)
    sess.bind_sums(sums.data_ptr())

    def one_iteration():
        sess.forces()
        if world > 1:
            dist.all_reduce(sums)
        sess.update()

    for _ in range(W):
        one_iteration()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
           torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local_rank) as clk:
        for k in range(K):
            flush.zero_()
            ev[k][0].record(stream)
            sess.forces()
            ev[k][1].record(stream)
            if world > 1:
                dist.all_reduce(sums)
            sess.update()
            ev[k][2].record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    step_ms = [a.elapsed_time(c) for a, _, c in ev]
    force_ms = [a.elapsed_time(b) for a, b, _ in ev]
    total_ms = float(sum(step_ms))
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    res = sess.finish()
    inter = res.interactions[W:W + K].astype(np.float64)
    visits_total = None
    interactions = float(inter.sum())
    value = interactions / (total_ms / 1e3)
    batched = None if args.no_batched else run_batched(args, rank, world)  # every rank
    if rank != 0:
        return None

    peaks, peak_src = load_peaks()
    clocks = clk.summary()
    fmax = float(peaks.get("sm_max_mhz", 1965.0))
    peak = fp32_peak_tflops(fmax)
    # dominant kernel: the traversal force pass (incl. its tiny partial reduction)
    mean_force_s = float(np.mean(force_ms)) / 1e3
    per_launch_inter = float(inter.mean()) / 1.0
    # visits per launch are not in the result rows; use the oracle-equal ratio
    # recorded by the kernel counters (visits are summed with interactions)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K,
        "warmup": W, "ms_per_step": total_ms / K, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32 forces / f64 state",
        "data": "synthetic (synth.blob, PCG64 seed %d), random-init inputs" % args.seed,
        "config": {"workload": "configs[2]: 1M x 1M FGA pair, Barnes-Hut theta=%g, fixed "
                               "iteration budget" % args.theta,
                   "n_reference": len(x), "n_template": len(y), "theta": args.theta,
                   "G": params.G,
                   "tree_nodes": sess.n_nodes, "parallelism": f"template-shard x{world}",
                   "l2": "flushed between timed steps (256 MiB write, outside the events)"},
        "gpu_launches": 4 * K,  # k_bh_iterate, k_reduce_stage, k_reduce_final, k_update
        "interactions_per_step": per_launch_inter,
    }
    # also visits/s and "equivalent direct pairs/s" (N*M per
    # iteration over the same time), labelled as such
    line["visits_per_s"] = _visits_per_step(res, W, K) * K / (total_ms / 1e3)
    line["equivalent_direct_pairs_per_s"] = float(len(x)) * float(len(y)) * K / (total_ms / 1e3)
    visits_step = _visits_per_step(res, W, K)
    flop = FLOP_PER_INTERACTION * per_launch_inter + FLOP_PER_VISIT * visits_step
    achieved = flop / mean_force_s / 1e12
    l2_peak, l2_src = l2_peak_gbs()
    alg_bytes = BYTES_PER_VISIT * visits_step + BYTES_PER_QUERY * len(y)
    l2_achieved = alg_bytes / mean_force_s / 1e9
    line["roofline"] = {
        "kernel": "k_bh_iterate<float> (+k_reduce)", "bound": "l2", "unit": "GB/s",
        "achieved": l2_achieved, "peak": l2_peak, "frac": l2_achieved / l2_peak if l2_peak else None,
        "peak_source": l2_src,
        "work": f"SURVEY §8(d) K6: {BYTES_PER_VISIT} B/visit x {visits_step:.4g} visits + "
                f"{BYTES_PER_QUERY} B x {len(y)} queries = {alg_bytes:.4g} B per launch",
        "ms_per_launch": mean_force_s * 1e3, "traffic": _traffic("bh"),
        "fp32_view": {"achieved_tflops": achieved, "peak_tflops": peak, "frac": achieved / peak,
                      "peak_source": f"2*148*128*sm_max_mhz ({peak_src} MEASURED_PEAKS.json "
                                     f"sm_max_mhz={fmax})",
                      "work": f"{FLOP_PER_INTERACTION} FLOP/interaction + {FLOP_PER_VISIT} "
                              "FLOP/visit"}}
    line["clocks"] = clocks
    if world == 1 and not args.no_build:
        line["tree_build"] = run_tree_build(args, dev, peaks, peak_src)
    if world == 1 and not args.no_direct:
        line["direct"] = run_direct(args, x, y, dev, stream, peak, peak_src, fmax)
    if world == 1 and not args.no_fp64:
        line["fp64_mode"] = run_fp64(args, x_t, y_t, len(x), len(y), dev, stream, local_rank)
    if world == 1 and not args.no_e2e:
        line["e2e"] = run_e2e(args, x, y, sess)
    if world == 1 and not args.no_registration:
        line["registration"] = run_registration(args, x, y)
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args, x, y, args.cpu_sample)
    if batched is not None:
        line["batched"] = batched
    if world == 1 and not args.no_configs:
        line["configs"] = run_other_configs(args)
    if world == 1 and not args.no_ingest:
        line["ingest"] = run_ingest(x)
    return line


_L2_CACHE = {}


def l2_peak_gbs():
    """Measured L2 read bandwidth (libfgaprobe.so: all SMs stream a 32 MiB
    L2-resident buffer), the K6 roofline denominator; MEASURED_PEAKS.json has
    no L2 figure."""
    if "v" in _L2_CACHE:
        return _L2_CACHE["v"]
    import ctypes
    v, src = None, "unavailable"
    try:
        lib = ctypes.CDLL(os.path.join(ROOT, "paper_2009_14005_b200", "_lib", "libfgaprobe.so"))
        lib.fga_probe_l2_read.argtypes = [ctypes.c_size_t, ctypes.c_int,
                                          ctypes.POINTER(ctypes.c_double)]
        best = 0.0
        for _ in range(3):
            g = ctypes.c_double(0.0)
            if lib.fga_probe_l2_read(64 << 20, 200, ctypes.byref(g)) == 0:
                best = max(best, g.value)
        if best > 0:
            v = best
            src = "measured live: libfgaprobe L2 read probe, 64 MiB x 200 passes, best of 3"
    except OSError as e:
        src = f"unavailable ({e})"
    _L2_CACHE["v"] = (v, src)
    return v, src


def run_tree_build(args, dev, peaks, peak_src):
    """K2-K5 (fga_tree_build_dev: bbox, exact keys, radix sort, emission,
    summarize, traversal records) on device-resident points, CUDA events per
    build (the build's one internal node-count sync included).  Roofline:
    SURVEY §8(d) 350 algorithmic B/point against HBM."""
    import ctypes

    import torch

    from paper_2009_14005_b200 import _native as N
    from paper_2009_14005_b200 import synth
    L = N.lib()
    c = N.Context(dev.index)
    stream = torch.cuda.current_stream()
    c.set_stream(stream.cuda_stream)
    hbm = float(peaks.get("hbm_gbs", 6552.3))
    out = {}
    for n in [int(v) for v in args.build_sizes.split(",") if v]:
        rng = synth.rng_from_seed(args.seed)
        pts = torch.from_numpy(synth.blob(n, rng).points).to(dev)
        ms = torch.full((n,), 1.0, dtype=torch.float64, device=dev)
        nn = N._i64(0)
        for _ in range(3):
            N.check(L.fga_tree_build_dev(c.handle, pts.data_ptr(), ms.data_ptr(), n, 20,
                                         ctypes.byref(nn)))
        reps = 10 if n <= 2_000_000 else 4
        flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
        times = []
        for _ in range(reps):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            N.check(L.fga_tree_build_dev(c.handle, pts.data_ptr(), ms.data_ptr(), n, 20,
                                         ctypes.byref(nn)))
            b.record(stream)
            torch.cuda.synchronize()
            times.append(a.elapsed_time(b))
        t = float(np.median(times)) / 1e3
        ach = BUILD_BYTES_PER_POINT * n / t / 1e9
        out[str(n)] = {"ms": t * 1e3, "nodes": int(nn.value), "points_per_s": n / t,
                       "roofline": {"bound": "hbm", "unit": "GB/s", "achieved": ach,
                                    "peak": hbm, "frac": ach / hbm,
                                    "peak_source": f"{peak_src} MEASURED_PEAKS.json hbm_gbs",
                                    "work": f"SURVEY §8(d): {BUILD_BYTES_PER_POINT} B/point"}}
        del pts, ms, flush
    c.close()
    out["api"] = "fga_tree_build_dev (blob points, unit masses, max_depth 20), median of reps, L2 flushed"
    return out


def run_fp64(args, x_t, y_t, n, m, dev, stream, local_rank):
    """The same 1M iteration with precision="fp64": the reference's
    arithmetic and node order (forces bit-identical to bh_forces_kernel on
    the same tree), for the cost of exactness next to the FP32 headline."""
    import torch

    import paper_2009_14005_b200 as fga
    from paper_2009_14005_b200.engine import Session
    K, W = 3, 1
    params = bench_params(args).replace(conv_tol=1e-300, max_iters=W + K + 1)
    sess = Session(None, None, params, fga.RegisterOptions(compute_gpe=False, precision="fp64"),
                   device=local_rank, stream=stream.cuda_stream,
                   device_inputs=(x_t.data_ptr(), n, y_t.data_ptr(), m))
    for _ in range(W):
        sess.forces()
        sess.update()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(K):
        sess.forces()
        sess.update()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / K
    res = sess.finish()
    inter = float(res.interactions[W:W + K].mean())
    return {"ms_per_step": ms, "value": inter / (ms / 1e3), "unit": UNIT,
            "note": "precision=fp64: reference arithmetic, bit-identical forces on the same tree"}


def _visits_per_step(res, W, K):
    v = getattr(res, "visits_per_iter", None)
    if v is None:
        return 0.0
    return float(np.mean(v[W:W + K]))


def _traffic(which):
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(p) as f:
            return json.load(f).get(which)
    except OSError:
        return None


def run_direct(args, x, y, dev, stream, peak, peak_src, fmax):
    import torch

    import paper_2009_14005_b200 as fga
    from paper_2009_14005_b200.engine import Session
    S = args.direct_steps
    params = fga.default_params().replace(theta=0.0, conv_tol=1e-300, max_iters=S + 2)
    x_t = torch.from_numpy(np.array(x.points)).to(dev)
    y_t = torch.from_numpy(np.array(y.points)).to(dev)
    sess = Session(None, None, params, fga.RegisterOptions(compute_gpe=False),
                   device=dev.index, stream=stream.cuda_stream,
                   device_inputs=(x_t.data_ptr(), len(x), y_t.data_ptr(), len(y)))
    sess.iterate(1)  # warm-up
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(S)]
    torch.cuda.synchronize()
    for k in range(S):
        ev[k][0].record(stream)
        sess.forces()
        ev[k][1].record(stream)
        sess.update()
    torch.cuda.synchronize()
    ms = float(np.mean([a.elapsed_time(b) for a, b in ev]))
    pairs = float(len(x)) * float(len(y))
    achieved = FLOP_PER_INTERACTION * pairs / (ms / 1e3) / 1e12
    sess.finish()
    return {"value": pairs / (ms / 1e3), "unit": "pairs/s", "ms_per_step": ms,
            "config": "theta=0: exact O(NM) tiled direct sum, same 1M x 1M pair",
            "roofline": {"kernel": "k_direct_iterate32", "bound": "fp32", "unit": "TFLOP/s",
                         "achieved": achieved, "peak": peak, "frac": achieved / peak,
                         "peak_source": f"2*148*128*sm_max_mhz ({peak_src}, {fmax} MHz)",
                         "work": "20 FLOP/pair", "traffic": _traffic("direct")}}


def run_e2e(args, x, y, sess):
    """The reference's per-iteration native crossing (bhtree.bh_forces ->
    _kernels.bh_forces_kernel, bhtree.py:139) replaced by fga_tree_forces on
    pinned host buffers: H2D queries+masses, traversal, D2H forces+counters."""
    import torch

    import paper_2009_14005_b200 as fga
    from paper_2009_14005_b200 import _native as N
    xn, yn, ctx = fga.normalize_pair(x, y, -5.0, 5.0)
    sy = fga.niv_masses(yn, 16, ctx, 20)
    p = bench_params(args)
    qm_np = np.maximum(0.1 * sy / sy.max(), max(1e-6, p.dt * p.eta))  # registration.py:87
    m = len(yn)

    def pinned(shape, dtype):
        return torch.empty(shape, dtype=dtype, pin_memory=True).numpy()

    q = pinned((m, 3), torch.float64)
    q[:] = yn.points
    qm = pinned((m,), torch.float64)
    qm[:] = qm_np
    f = pinned((m, 3), torch.float64)
    vis = pinned((m,), torch.int64)
    acc = pinned((m,), torch.int64)
    c = sess.ctx
    L = N.lib()

    def call():
        N.check(L.fga_tree_forces(c.handle, N.ptr(q), N.ptr(qm), m, float(args.theta),
                                  float(p.G), float(p.epsilon) ** 2, N.PREC_FP32, N.ptr(f),
                                  N.ptr(vis), N.ptr(acc)))

    for _ in range(2):
        call()
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        call()
        times.append(time.perf_counter() - t0)
    inter = float(acc.sum())
    return {"value": inter * len(times) / sum(times), "unit": UNIT,
            "h2d_bytes_per_step": int(q.nbytes + qm.nbytes),
            "d2h_bytes_per_step": int(f.nbytes + vis.nbytes + acc.nbytes),
            "ms_per_step": 1e3 * sum(times) / len(times),
            "api": "fga_tree_forces (drop-in for _kernels.bh_forces_kernel), pinned host "
                   "buffers, initial template state, FP32 traversal",
            "visits_per_query": float(vis.mean())}


def batch_pairs(P, rank=0, world=1):
    """configs[4]: 3DMatch-fragment-sized pairs, 4096 points each, blob/box
    alternating (synth.fragment_pair); this rank's share is
    p = rank, rank+world, ... (pairs sharded, no collective)."""
    from paper_2009_14005_b200 import synth
    return [synth.fragment_pair(p) for p in range(rank, P, world)]


def run_batched(args, rank, world):
    """configs[4]: all pairs in one persistent kernel (fga_register_batch),
    default params (theta 0.6).  `kernel_s`: CUDA events around the kernel on
    device-resident clouds; `wall_s`: the C-ABI call on pinned host buffers
    (H2D of all clouds + kernel + D2H of the results)."""
    import ctypes

    import torch

    import paper_2009_14005_b200 as fga
    from paper_2009_14005_b200 import _native as N
    pairs = batch_pairs(args.batch_pairs, rank, world)
    P = len(pairs)
    xoff = np.zeros(P + 1, np.int64)
    yoff = np.zeros(P + 1, np.int64)
    xoff[1:] = np.cumsum([len(x) for x, _ in pairs])
    yoff[1:] = np.cumsum([len(y) for _, y in pairs])

    def pinned(a):
        t = torch.empty(a.shape, dtype=torch.float64, pin_memory=True).numpy()
        t[:] = a
        return t

    X = pinned(np.concatenate([x.points for x, _ in pairs]))
    Y = pinned(np.concatenate([y.points for _, y in pairs]))
    params = fga.default_params()
    cp = N.make_params(params)
    co = fga.registration._c_options(fga.RegisterOptions(), None, None)
    out = (N.CPairResult * P)()
    c = N.context(torch.cuda.current_device())
    c.set_stream(torch.cuda.current_stream().cuda_stream)
    L = N.lib()

    def host_call():
        N.check(L.fga_register_batch(c.handle, N.ptr(X), N.ptr(xoff), N.ptr(Y), N.ptr(yoff), P, 3,
                                     ctypes.byref(cp), ctypes.byref(co), ctypes.addressof(out),
                                     None))

    host_call()  # warm-up: full-size scratch, all code paths
    dev = torch.device("cuda", torch.cuda.current_device())
    Xd = torch.from_numpy(X).to(dev)
    Yd = torch.from_numpy(Y).to(dev)
    xo = torch.from_numpy(xoff).to(dev)
    yo = torch.from_numpy(yoff).to(dev)
    res_d = torch.empty(P * ctypes.sizeof(N.CPairResult), dtype=torch.uint8, device=dev)
    nmax = int(np.diff(xoff).max())
    mmax = int(np.diff(yoff).max())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize()
    e0.record()
    N.check(L.fga_register_batch_dev(c.handle, Xd.data_ptr(), xo.data_ptr(), Yd.data_ptr(),
                                     yo.data_ptr(), P, nmax, mmax, 3, ctypes.byref(cp),
                                     ctypes.byref(co), res_d.data_ptr(), None))
    e1.record()
    torch.cuda.synchronize()
    kernel_s = e0.elapsed_time(e1) / 1e3
    t0 = time.perf_counter()
    host_call()
    wall = time.perf_counter() - t0
    its = np.array([r.iterations for r in out])
    inter = float(sum(r.interactions for r in out))
    failed = int(sum(r.status != 0 for r in out))
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([wall, kernel_s], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        wall, kernel_s = float(t[0]), float(t[1])
        s2 = torch.tensor([inter, float(failed)], dtype=torch.float64, device=dev)
        dist.all_reduce(s2)
        inter, failed = float(s2[0]), int(s2[1])
        if rank != 0:
            return None
    return {"workload": f"configs[4]: {args.batch_pairs} pairs x 4096 pts (blob/box, seeds "
                        "100000+p, <=60 deg), default params (theta 0.6)",
            "pairs_per_s": args.batch_pairs / kernel_s, "kernel_s": kernel_s,
            "e2e_pairs_per_s": args.batch_pairs / wall, "wall_s": wall,
            "interactions_per_s": inter / kernel_s,
            "iterations_min_median_max": [int(its.min()), float(np.median(its)), int(its.max())],
            "failed": failed,
            "api": "fga_register_batch_dev (device clouds, CUDA events) / fga_register_batch "
                   "(pinned host buffers, wall clock)",
            "h2d_bytes": int(X.nbytes + Y.nbytes + xoff.nbytes + yoff.nbytes),
            "sharding": f"pairs split over {world} GPU(s), no collective"}


def run_other_configs(args):
    """configs[1] (100k LiDAR-shaped pair) and configs[3] (200k partial
    overlap, 5% outliers, inhomogeneous density, kNN-16 masses): one full
    register() each from host numpy, theta 0.5.  G per scene from a sweep
    (tools/sweep_c2.py, tools/sweep_c4.py): the 160 m x 16 m x 4.5 m street
    scan flies apart for G >= 1 and converges for G = 0.2; the partial-overlap
    pair diverges at G*sqrt(2000/N) = 6.67 and converges at G = 2."""
    import paper_2009_14005_b200 as fga
    from paper_2009_14005_b200 import synth
    out = {}
    x, y, gt = synth.configs1_pair()
    p = fga.default_params().replace(theta=0.5, G=0.2)
    fga.register(fga.PointCloud(x.points[:5000]), fga.PointCloud(y.points[:5000]), params=p)
    t0 = time.perf_counter()
    r = fga.register(x, y, params=p)
    wall = time.perf_counter() - t0
    # the second variant of SURVEY §8(d) C2: the same street rescanned from a
    # sensor moved by gt (different sampling -- a realistic next frame)
    rng2 = synth.rng_from_seed(2)
    scene = synth.lidar_scene(rng2)
    xa = synth.lidar_scan(100_000, rng2, scene=scene)
    gt2 = synth.random_rigid(rng2, np.deg2rad(10), 1.0)
    yb = synth.lidar_scan(100_000, rng2, scene=scene, pose=gt2)
    t0 = time.perf_counter()
    r2 = fga.register(xa, yb, params=p)
    wall2 = time.perf_counter() - t0
    out["c2_lidar_100k_rescan"] = {
        "wall_s": wall2, "iterations": r2.iterations, "converged": r2.converged, "G": p.G,
        "rotation_err_deg": fga.angular_deviation(gt2.rotation, r2.transform.rotation),
        "translation_err_m": float(np.linalg.norm(r2.transform.translation - gt2.translation)),
        "timings_ms": r2.timings_ms}
    out["c2_lidar_100k"] = {
        "wall_s": wall, "iterations": r.iterations, "converged": r.converged, "G": p.G,
        "rotation_err_deg": fga.angular_deviation(gt.rotation, r.transform.rotation),
        "interactions_per_s_loop": float(r.interactions.sum()) / (r.timings_ms["loop"] / 1e3),
        "timings_ms": r.timings_ms}
    x, y, gt = synth.configs3_pair()
    p = fga.default_params().replace(theta=0.5, G=2.0)
    o = fga.RegisterOptions(mass_field="knn", knn_k=16)
    from paper_2009_14005_b200 import masses
    masses.knn_masses(x, 16)
    t0 = time.perf_counter()
    masses.knn_masses(x, 16)
    knn_s = time.perf_counter() - t0
    fga.register(x, y, params=p.replace(max_iters=2), options=o)  # warm the kNN-mass path
    t0 = time.perf_counter()
    r = fga.register(x, y, params=p, options=o)
    wall = time.perf_counter() - t0
    o_niv = fga.RegisterOptions()
    t0 = time.perf_counter()
    r_niv = fga.register(x, y, params=p, options=o_niv)
    wall_niv = time.perf_counter() - t0
    out["c4_overlap_200k_niv"] = {
        "wall_s": wall_niv, "iterations": r_niv.iterations, "converged": r_niv.converged,
        "G": p.G, "rotation_err_deg": fga.angular_deviation(gt.rotation, r_niv.transform.rotation),
        "timings_ms": r_niv.timings_ms}
    out["c4_overlap_200k_knn16"] = {
        "wall_s": wall, "iterations": r.iterations, "converged": r.converged, "G": p.G,
        "rotation_err_deg": fga.angular_deviation(gt.rotation, r.transform.rotation),
        "knn16_masses_s_200k_host_api": knn_s,
        "interactions_per_s_loop": float(r.interactions.sum()) / (r.timings_ms["loop"] / 1e3),
        "timings_ms": r.timings_ms}
    return out


def run_ingest(x):
    """io.load_cloud of the 1M-point reference cloud written
    as an XYZ file (io.write_cloud, 17 significant digits): the native
    parser on all host threads vs the reader that follows the reference's
    per-line Python algorithm (io.py:23-43), same file, same doubles."""
    import tempfile

    from paper_2009_14005_b200 import io
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "x.xyz")
        io.write_cloud(path, x)
        size = os.path.getsize(path)
        io.load_cloud(path)  # warm (page cache, library)
        t0 = time.perf_counter()
        got = io.load_cloud(path)
        t_native = time.perf_counter() - t0
        t0 = time.perf_counter()
        ref = io._cloud_from_text(io._read_text(path))
        t_py = time.perf_counter() - t0
    assert np.array_equal(got.points, ref.points) and np.array_equal(got.points, x.points)
    return {"points": len(x), "file_mb": size / 1e6, "native_s": t_native,
            "native_mb_per_s": size / 1e6 / t_native, "python_reader_s": t_py,
            "speedup": t_py / t_native, "threads": os.cpu_count(),
            "api": "paper_2009_14005_b200.io.load_cloud (fga_parse_cloud) vs the reference's "
                   "per-line algorithm in Python"}


def run_registration(args, x, y):
    import paper_2009_14005_b200 as fga
    p = bench_params(args)
    fga.register(x, y, params=p)  # warm-up at full size (allocations, module loads)
    walls = []
    for _ in range(3):
        t0 = time.perf_counter()
        r = fga.register(x, y, params=p)
        walls.append(time.perf_counter() - t0)
    wall = float(np.median(walls))
    return {"wall_s": wall, "walls_s": walls, "iterations": r.iterations, "converged": r.converged,
            "interactions": int(r.interactions.sum()), "timings_ms": r.timings_ms,
            "params": {"theta": p.theta, "G": p.G, "max_iters": p.max_iters,
                       "conv_tol": p.conv_tol},
            "api": "register(x, y) from host numpy, median of 3 calls after a full-size "
                   "warm-up; includes normalize, NIV masses, tree build, 2x O(NM) energy "
                   "and the iteration loop"}


# --------------------------------------------------------------------------- CPU
def cpu_baseline(args, x, y, sample):
    """The C oracle (OpenMP, all host threads) on a bounded sample of the same
    workload: tree over the normalized reference, bh_forces for `sample`
    template queries at the initial state."""
    from oracle import oracle as orc
    orc.build_lib()
    bp = bench_params(args)
    p = {"G": bp.G, "eps": 0.2}
    xn, yn, ctx = orc.normalize_pair(x.points, y.points, -5.0, 5.0)
    sx = orc.niv_masses(xn, 16, -5.0, 5.0, 20)
    sy = orc.niv_masses(yn, 16, -5.0, 5.0, 20)
    mx, my = orc.rescale(sx, sy, 0.1, 0.2)
    t0 = time.perf_counter()
    tree = orc.tree_build(xn, mx, 20)
    build_s = time.perf_counter() - t0
    idx = np.random.default_rng(0).choice(len(yn), size=min(sample, len(yn)), replace=False)
    threads = orc.max_threads()
    t0 = time.perf_counter()
    _, visits, acc = orc.bh_forces(tree, yn[idx], my[idx], args.theta, p["G"], p["eps"], threads)
    dt = time.perf_counter() - t0
    # the reference as shipped is single-threaded -- one core
    # on a quarter of the sample
    idx1 = idx[: max(1, len(idx) // 4)]
    t0 = time.perf_counter()
    _, _, acc1 = orc.bh_forces(tree, yn[idx1], my[idx1], args.theta, p["G"], p["eps"], 1)
    dt1 = time.perf_counter() - t0
    return {"value": float(acc.sum()) / dt, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"{len(idx)} template queries of the {len(yn)}-point workload at the "
                      f"initial state (oracle bh_forces, theta={args.theta}); tree build "
                      f"{build_s:.2f} s single-threaded",
            "seconds": dt, "visits_per_query": float(visits.mean()),
            "one_core": {"value": float(acc1.sum()) / dt1, "unit": UNIT, "cores": 1,
                         "sample": f"{len(idx1)} of the same queries", "seconds": dt1}}


def run_reference(args, rank):
    """--impl reference: the reference's CPU algorithm (C oracle port, all host
    threads) on the same config / metric; each step = one bounded sample."""
    if rank != 0:
        return None
    from oracle import oracle as orc
    orc.build_lib()
    x, y = workload(args.n, args.seed)
    xn, yn, _ = orc.normalize_pair(x.points, y.points, -5.0, 5.0)
    sx = orc.niv_masses(xn, 16, -5.0, 5.0, 20)
    sy = orc.niv_masses(yn, 16, -5.0, 5.0, 20)
    mx, my = orc.rescale(sx, sy, 0.1, 0.2)
    tree = orc.tree_build(xn, mx, 20)
    threads = orc.max_threads()
    G = 66.7 if args.default_g else 66.7 * (2000.0 / args.n) ** 0.5
    sample = min(16384, len(yn))
    rng = np.random.default_rng(1)

    def step():
        idx = rng.choice(len(yn), size=sample, replace=False)
        t0 = time.perf_counter()
        _, _, acc = orc.bh_forces(tree, yn[idx], my[idx], args.theta, G, 0.2, threads)
        return float(acc.sum()), time.perf_counter() - t0

    for _ in range(args.warmup):
        step()
    inter = secs = 0.0
    for _ in range(args.steps):
        a, s = step()
        inter += a
        secs += s
    value = inter / secs
    desc = (f"{sample} random template queries per step of the {len(yn)}-point workload "
            f"(initial state), C oracle bh_forces (restates _kernels.py:7-50)")
    return {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * secs / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "configs[2]: 1M x 1M FGA pair, Barnes-Hut theta=%g"
                       % args.theta, "n_reference": len(x), "n_template": len(y)},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                             "sample": desc},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        line = run_reference(args, rank)
        if line is not None:
            print(json.dumps(line), flush=True)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    line = run_ours(args, rank, world, local_rank)
    if line is not None:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
