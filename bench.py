#!/usr/bin/env python
"""FGA hot-path benchmark on B200 (contract: see DESIGN.md "Measurement").

Workload (BASELINE.json configs[2], the 1M-point FGA the metric is quoted
on): a 1,000,000 x 1,000,000 synthetic blob pair (synth.configs2_pair, PCG64
seed 3, random rotation <= 60 deg, translation <= 0.1), Barnes-Hut theta =
0.5.  A "step" is one FGA iteration at the INITIAL template state (SURVEY
§8(d): the headline interactions/s is quoted at iteration 0): the force pass
over the whole template (traversal + fused Euler-Cromer step + Kabsch
partials), the partial reduction (+ the all-reduce for N > 1) and the fp64
rigid update; the state is restored on the device (fga_session_checkpoint)
before every step, outside the timed region.  `value` = accepted
particle-node interactions per second (each accepted node is one softened
pair interaction, the reference's own unit: _kernels.py:37-42), whole job.

The reference arm (--impl reference) times the oracle port of the reference's
CPU path on the same config and the same state (sampled queries), on all
host cores.

Extra legs on the same JSON line (N=1 unless noted): `e2e` (the reference-
facing bh_forces drop-in with pinned host buffers, every rank its query
share), `fp64_mode`, `direct` (theta = 0, exact O(NM)), `gpe` (the O(NM)
energy), `small_m` (shard 0 of 8 on one GPU), `tree_build`, `registration`
(full register() wall time, with the CPU reference extrapolated beside it),
`configs0` (configs[0] register() on GPU vs the oracle on 1 and all host
cores, measured), `batched` (configs[4], pairs sharded over ranks),
`configs` (configs[1]/[3]), `ingest`, `cpu_baseline`.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    python bench.py --gpus 2 --dry-run      # CPU/gloo plumbing check
Without WORLD_SIZE in the environment, --gpus N > 1 re-launches itself under
torch.distributed.run with N ranks (127.0.0.1).
"""

from __future__ import annotations

import argparse
import json
import os
import socket
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
KERNELS_PER_STEP = 6       # k_qbound, k_node_bands, k_bh_iterate, k_reduce_stage/_final, k_update


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=1_000_000)
    ap.add_argument("--theta", type=float, default=0.5)
    ap.add_argument("--seed", type=int, default=3)
    ap.add_argument("--dry-run", action="store_true",
                    help="CPU only: exercise the launch / rank / barrier / max-over-ranks "
                         "plumbing with gloo and print the JSON line")
    for leg in ("direct", "e2e", "registration", "cpu-baseline", "batched", "build", "fp64",
                "ingest", "configs", "gpe", "small-m", "configs0"):
        ap.add_argument(f"--no-{leg}", action="store_true")
    ap.add_argument("--direct-steps", type=int, default=3)
    ap.add_argument("--build-sizes", default="1000000,16000000")
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


def config_dict(args, n_ref, n_tpl, tree_nodes, world):
    """The workload description, identical in both arms."""
    p = bench_params(args)
    return {"workload": "configs[2]: 1M x 1M FGA pair, Barnes-Hut theta=%g, one iteration "
                        "at the initial template state" % args.theta,
            "n_reference": int(n_ref), "n_template": int(n_tpl), "theta": args.theta,
            "G": p.G, "epsilon": p.epsilon, "seed": args.seed, "tree_nodes": int(tree_nodes),
            "state": "initial template state (iteration 0), restored before every step",
            "parallelism": f"template-shard x{world}",
            "l2": "flushed between timed steps (256 MiB write, outside the events)"}


def host_threads():
    """Host threads for the CPU legs: every core this process may run on,
    passed explicitly to the oracle's OpenMP regions (torch.distributed.run
    sets OMP_NUM_THREADS=1 in every rank, which would otherwise leave the
    reference arm on one core at N > 1)."""
    try:
        return len(os.sched_getaffinity(0))
    except (AttributeError, OSError):
        return os.cpu_count() or 1


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0}, "fallback"


def fp32_peak_tflops(sm_mhz, sms=148):
    return 2.0 * sms * 128 * sm_mhz * 1e6 / 1e12


def _profile(which):
    """Per-launch counters of the hot kernels from the committed ncu capture
    (profiles/traffic.json, tools/profile_kernels.sh + tools/ncu_metrics.py)."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(p) as f:
            return json.load(f).get(which) or {}
    except OSError:
        return {}


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def relaunch(args):
    """--gpus N without WORLD_SIZE: run this script under torch.distributed.run
    with N ranks on this node (rank 0 prints the JSON line)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(_free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def run_dry(args, rank, world):
    """The multi-rank plumbing without a GPU: gloo process group, W untimed and
    K timed steps bracketed by barriers, max over ranks of the step time, one
    JSON line from rank 0 (tests/test_bench_plumbing.py)."""
    import torch
    import torch.distributed as dist
    if world > 1:
        dist.init_process_group("gloo")
    work = np.random.default_rng(rank).normal(size=(200_000,))

    def step():
        return float(np.sort(work)[0])

    for _ in range(args.warmup):
        step()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    if world > 1:
        dist.barrier()
    dt = time.perf_counter() - t0
    t = torch.tensor([dt], dtype=torch.float64)
    n = torch.tensor([float(len(work) * args.steps)], dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(n)
    if world > 1:
        dist.destroy_process_group()
    if rank != 0:
        return None
    return {"metric": METRIC, "value": float(n.item()) / float(t.item()), "unit": "elements/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * float(t.item()) / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "dry_run": True, "ranks_reporting": world,
            "config": {"workload": "dry run: CPU sort per rank (plumbing check only)"}}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region
    (samples are matched to the region by their timestamps)."""

    FIELDS = ("timestamp,clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = os.path.join("/tmp", f"fga_clocks_{os.getpid()}.csv")
        self.t0 = self.t1 = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        # nvidia-smi takes a few hundred ms to start: the region begins once
        # it is sampling
        t_end = time.time() + 5.0
        while self.proc is not None and time.time() < t_end and not self._rows():
            time.sleep(0.02)
        self.t0 = time.time()
        return self

    def _rows(self):
        try:
            rows = [r.split(",") for r in open(self.path).read().strip().splitlines()]
        except OSError:
            return []
        return [[c.strip() for c in r] for r in rows if len(r) >= 8]

    def __exit__(self, *a):
        self.t1 = time.time()
        if self.proc is not None:
            time.sleep(0.15)
            self.proc.terminate()
            self.proc.wait()

    @staticmethod
    def _ts(v):
        import datetime
        try:
            return datetime.datetime.strptime(v, "%Y/%m/%d %H:%M:%S.%f").timestamp()
        except ValueError:
            return None

    def summary(self):
        rows = self._rows()
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        stamped = [(self._ts(r[0]), r) for r in rows]
        inside = [r for t, r in stamped if t is not None and self.t0 - 0.06 <= t <= self.t1 + 0.06]
        if not inside:  # (a region shorter than the sampling period) the nearest sample
            mid = 0.5 * (self.t0 + self.t1)
            inside = [min(stamped, key=lambda tr: abs((tr[0] or 0.0) - mid))[1]]
        sm = [float(r[1]) for r in inside if r[1].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in inside:
            for nm, v in zip(names, r[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": float(inside[0][2]) if inside[0][2].replace(".", "").isdigit() else None,
                "reasons": sorted(reasons), "samples": len(inside),
                "region_s": round(self.t1 - self.t0, 3)}


# --------------------------------------------------------------------------- ours
def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    import paper_2009_14005_b200 as fga
    from paper_2009_14005_b200.engine import SUM_VISITS, SUMS_LEN, Session

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    x, y = workload(args.n, args.seed)
    K, W = args.steps, args.warmup
    params = bench_params(args).replace(conv_tol=1e-300, max_iters=4)
    x_t = torch.from_numpy(np.array(x.points)).to(dev)
    y_t = torch.from_numpy(np.array(y.points)).to(dev)
    stream = torch.cuda.current_stream()

    from paper_2009_14005_b200 import _native as N

    def session(count_visits=False, precision="fp32", shard=(rank, world)):
        # one context per session: a context holds one registration session
        s = Session(None, None, params,
                    fga.RegisterOptions(compute_gpe=False, count_visits=count_visits,
                                        precision=precision),
                    shard_rank=shard[0], shard_count=shard[1], device=local_rank,
                    stream=stream.cuda_stream,
                    device_inputs=(x_t.data_ptr(), len(x), y_t.data_ptr(), len(y)),
                    ctx=N.Context(local_rank))
        sums = torch.zeros(SUMS_LEN, dtype=torch.float64, device=dev)
        s.bind_sums(sums.data_ptr())
        s.checkpoint()  # the initial state: every step starts from it
        return s, sums

    sess, sums = session()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2

    def one_step(ev=None):
        sess.restore()
        flush.zero_()
        if ev:
            ev[0].record(stream)
        sess.forces()
        if ev:
            ev[1].record(stream)
        if world > 1:
            dist.all_reduce(sums)
        sess.update()
        if ev:
            ev[2].record(stream)

    for _ in range(W):
        one_step()
    ev = [tuple(torch.cuda.Event(enable_timing=True) for _ in range(3)) for _ in range(K)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local_rank) as clk:
        for k in range(K):
            one_step(ev[k])
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    step_ms = [a.elapsed_time(c) for a, _, c in ev]
    force_ms = [a.elapsed_time(b) for a, b, _ in ev]
    t = torch.tensor([float(sum(step_ms))], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    res = sess.finish()
    inter = float(res.interactions[0])  # all-reduced: the whole job's count per step
    value = inter * K / (total_ms / 1e3)
    # node visits of the same state (an untimed counting pass; identical
    # traversal, visits are not counted in the timed kernel)
    vsess, vsums = session(count_visits=True)
    vsess.forces()
    if world > 1:
        dist.all_reduce(vsums)
    torch.cuda.synchronize()
    visits = float(vsums[SUM_VISITS].item())
    vsess.finish()
    del vsess
    tree_nodes = sess.n_nodes
    e2e = None if args.no_e2e else run_e2e(args, x, y, rank, world, local_rank)
    batched = None if args.no_batched else run_batched(args, rank, world)
    if rank != 0:
        return None

    peaks, peak_src = load_peaks()
    clocks = clk.summary()
    fmax = float(peaks.get("sm_max_mhz", 1965.0))
    peak = fp32_peak_tflops(fmax)
    mean_force_s = float(np.mean(force_ms)) / 1e3
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K,
        "warmup": W, "ms_per_step": total_ms / K, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32 forces / f64 state",
        "data": "synthetic (synth.configs2_pair, PCG64 seed %d), random-init inputs" % args.seed,
        "config": config_dict(args, len(x), len(y), tree_nodes, world),
        "gpu_launches": KERNELS_PER_STEP * K,
        "interactions_per_step": inter, "visits_per_step": visits,
        "visits_per_s": visits * K / (total_ms / 1e3),
        "equivalent_direct_pairs_per_s": float(len(x)) * float(len(y)) * K / (total_ms / 1e3),
    }
    if e2e is not None:
        line["e2e"] = e2e
    line["roofline"] = traversal_roofline(mean_force_s, visits, inter, len(y), peak, peak_src,
                                          fmax)
    line["clocks"] = clocks
    if world == 1 and not args.no_small_m:
        line["small_m"] = run_small_m(args, session, inter, mean_force_s, len(y))
    if world == 1 and not args.no_fp64:
        line["fp64_mode"] = run_fp64(session, stream, inter)
    if world == 1 and not args.no_gpe:
        line["gpe"] = run_gpe(session, stream, len(x), len(y), peak, peak_src, fmax)
    del sess
    torch.cuda.empty_cache()
    if world == 1 and not args.no_build:
        line["tree_build"] = run_tree_build(args, dev, peaks, peak_src)
    if world == 1 and not args.no_direct:
        line["direct"] = run_direct(args, x, y, dev, stream, peak, peak_src, fmax)
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args, x, y, args.cpu_sample)
        line["cpu_baseline"] = cpu
        if "fp64_mode" in line:
            line["fp64_mode"]["vs_cpu_baseline"] = line["fp64_mode"]["value"] / cpu["value"]
        line["vs_cpu_baseline"] = {"value": value / cpu["value"],
                                   "e2e": (e2e["value"] / cpu["value"]) if e2e else None,
                                   "note": "GPU arm / oracle port on all host cores, same "
                                           "state; the driver computes its own ratio"}
    if world == 1 and not args.no_registration:
        line["registration"] = run_registration(args, x, y, cpu)
    if world == 1 and not args.no_configs0:
        line["configs0"] = run_configs0()
    if batched is not None:
        line["batched"] = batched
    if world == 1 and not args.no_configs:
        line["configs"] = run_other_configs(args)
    if world == 1 and not args.no_ingest:
        line["ingest"] = run_ingest(x)
    return line


def traversal_roofline(force_s, visits, inter, m, peak_tflops, peak_src, fmax):
    """k_bh_iterate is issue-bound inside the SM (ncu: issue slots ~80% busy,
    a latency chain of warp-uniform L1-hit record loads), not a DRAM or
    tensor kernel, so the headline roofline is the issue-slot one: warp
    instructions per launch (ncu, profiles/traffic.json) / the live launch
    time, against 148 SMs x 4 schedulers x f_max.  Beside it: the SURVEY
    §8(d) byte model (32 B per query-node visit + 32 B per query) against the
    live-measured L2 read bandwidth -- it counts the L1 hits as traffic, so
    its fraction can exceed 1 -- with the L2->SM and DRAM bytes ncu measured
    per launch as `traffic`, and an FP32 FLOP view."""
    prof = _profile("bh")
    l2_peak, l2_src = l2_peak_gbs()
    alg = BYTES_PER_VISIT * visits + BYTES_PER_QUERY * m
    ach = alg / force_s / 1e9
    flop = FLOP_PER_INTERACTION * inter + FLOP_PER_VISIT * visits
    l2_view = {"unit": "GB/s", "achieved": ach, "peak": l2_peak,
               "frac": ach / l2_peak if l2_peak else None, "peak_source": l2_src,
               "work": f"SURVEY §8(d) K6: {BYTES_PER_VISIT} B/visit x {visits:.4g} visits + "
                       f"{BYTES_PER_QUERY} B x {m} queries = {alg:.4g} B per launch (model "
                       "bytes: most node loads are L1 hits, so frac may exceed 1)"}
    fp32_view = {"achieved_tflops": flop / force_s / 1e12, "peak_tflops": peak_tflops,
                 "frac": flop / force_s / 1e12 / peak_tflops,
                 "peak_source": f"2*148*128*sm_max_mhz ({peak_src} {fmax} MHz)",
                 "work": f"{FLOP_PER_INTERACTION} FLOP/interaction + {FLOP_PER_VISIT} FLOP/visit"}
    out = {"kernel": "k_bh_iterate<float> (+k_qbound, k_node_bands, k_reduce)",
           "ms_per_launch": force_s * 1e3,
           "traffic": prof.get("dram_bytes"),
           "traffic_source": "ncu dram__bytes_read.sum + dram__bytes_write.sum per launch, "
                             "profiles/traffic.json",
           "l2_to_sm_bytes": prof.get("lts_bytes"), "l1_hit_pct": prof.get("l1_hit_pct"),
           "l2_model_view": l2_view, "fp32_view": fp32_view}
    if prof.get("inst_executed"):
        issue_peak = 148 * 4 * fmax * 1e6  # warp-instructions per second
        achieved = prof["inst_executed"] / force_s
        out.update({"bound": "issue (latency-bound L1 record loads; not DRAM or tensor)",
                    "unit": "warp-inst/s", "achieved": achieved, "peak": issue_peak,
                    "frac": achieved / issue_peak,
                    "peak_source": f"148 SMs x 4 schedulers x {fmax} MHz",
                    "work": f"{prof['inst_executed']:.4g} warp instructions per launch (ncu)",
                    "ncu_issue_active_pct": prof.get("issue_active_pct"),
                    "ncu_warps_active_pct": prof.get("warps_active_pct")})
    else:
        out.update({"bound": "issue/L1TEX (no ncu profile: the byte model)", **l2_view})
    return out


def run_small_m(args, session, inter_full, force_s_full, m_full):
    """Shard 0 of 8 (M/8 = 125k queries, the per-GPU share of the 8-GPU
    strong-scaling run) on one GPU: its per-query interaction rate against
    the full 1M pass's."""
    import torch

    from paper_2009_14005_b200.engine import SUM_ACCEPTED
    s, sums = session(shard=(0, 8))
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=sums.device)
    times, inter = [], 0.0
    for k in range(8):
        s.restore()
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        s.forces()
        b.record(stream)
        torch.cuda.synchronize()
        inter = float(sums[SUM_ACCEPTED].item())
        s.update()
        if k >= 2:
            times.append(a.elapsed_time(b) / 1e3)
    m_local = s.m_local
    s.finish()
    t = float(np.mean(times))
    full = inter_full / force_s_full
    return {"queries": m_local, "ms_per_pass": t * 1e3, "interactions_per_s": inter / t,
            "interactions_per_s_vs_1m": inter / t / full,
            "ideal_ms": force_s_full * 1e3 * inter / inter_full,
            "note": "shard 0 of 8 of the configs[2] template (fga_session shard_rank=0, "
                    "shard_count=8), force pass at the initial state, CUDA events; the "
                    "passes after the first (which records the warps' node traces) run as "
                    "split passes (forces.cu k_bh_split)"}


def run_fp64(session, stream, inter32):
    """The same step with precision="fp64": the reference's arithmetic and
    node order (forces bit-identical to bh_forces_kernel on the same tree)."""
    import torch
    s, sums = session(precision="fp64")
    times = []
    for k in range(4):
        s.restore()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        s.forces()
        s.update()
        b.record(stream)
        torch.cuda.synchronize()
        if k:
            times.append(a.elapsed_time(b))
    res = s.finish()
    ms = float(np.mean(times))
    inter = float(res.interactions[0])
    return {"ms_per_step": ms, "value": inter / (ms / 1e3), "unit": UNIT,
            "same_accepted_set_as_fp32": inter == inter32,
            "note": "precision=fp64: reference arithmetic, bit-identical forces on the same "
                    "tree; same initial state"}


def run_gpe(session, stream, n, m, peak, peak_src, fmax):
    """The O(NM) energy (_kernels.py:53-67, k_gpe32: FP32 pairs, fp64 across
    tiles) of the initial template vs the 1M reference -- twice per
    register(), its largest cost."""
    import torch
    prof = _profile("gpe")
    sess, _ = session()
    times = []
    for k in range(3):
        sess.restore()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        sess.gpe()
        b.record(stream)
        torch.cuda.synchronize()
        sess.take_gpe()
        if k:
            times.append(a.elapsed_time(b) / 1e3)
    sess.finish()
    t = float(np.mean(times))
    pairs = float(n) * float(m)
    ach = FLOP_PER_INTERACTION * pairs / t / 1e12
    out = {"ms": t * 1e3, "pairs_per_s": pairs / t,
           "roofline": {"kernel": "k_gpe32", "bound": "FP32 FMA + MUFU", "unit": "TFLOP/s",
                        "achieved": ach, "peak": peak, "frac": ach / peak,
                        "peak_source": f"2*148*128*sm_max_mhz ({peak_src}, {fmax} MHz)",
                        "work": "20 FLOP-equivalent per pair (SURVEY §8(d) K11)",
                        "traffic": prof.get("dram_bytes"),
                        "ncu_fma_pipe_pct": prof.get("fma_pipe_pct"), "ncu_xu_pipe_pct": prof.get("xu_pipe_pct"),
                        "ncu_issue_active_pct": prof.get("issue_active_pct")}}
    return out


def run_e2e(args, x, y, rank, world, local_rank):
    """The reference's per-iteration native crossing (bhtree.bh_forces ->
    _kernels.bh_forces_kernel, bhtree.py:139) replaced by fga_tree_forces on
    pinned host buffers: H2D queries+masses, traversal, D2H forces+counters,
    inside the timed region.  Same state (initial template) and tree as the
    headline; with N ranks each evaluates its 1/N of the queries (max over
    ranks of the wall time, accepted interactions summed)."""
    import ctypes

    import torch
    import torch.distributed as dist

    import paper_2009_14005_b200 as fga
    from paper_2009_14005_b200 import _native as N
    from paper_2009_14005_b200 import bhtree
    xn, yn, ctx = fga.normalize_pair(x, y, -5.0, 5.0)
    p = bench_params(args)
    sx = fga.niv_masses(xn, 16, ctx, 20)
    sy = fga.niv_masses(yn, 16, ctx, 20)
    # registration.py:85-87 (the same mass fields the session builds)
    mx = np.minimum(16.0 * np.sqrt(len(sx) / 2000) * sx / sx.sum(), 0.022)
    my = np.maximum(0.1 * sy / sy.max(), max(1e-6, p.dt * p.eta))
    c = N.context(local_rank)
    bhtree.build(xn, mx, 20)  # the operator tree of this context (outside the timing)
    m = len(yn)
    L = N.lib()
    total = N._i64(0)

    def pinned(shape, dtype):
        return torch.empty(shape, dtype=dtype, pin_memory=True).numpy()

    def slice_calls(lo, hi, sync, with_visits=False):
        mm = hi - lo
        q = pinned((mm, 3), torch.float64)
        q[:] = yn.points[lo:hi]
        qm = pinned((mm,), torch.float64)
        qm[:] = my[lo:hi]
        f = pinned((mm, 3), torch.float64)
        vis = pinned((mm,), torch.int64)

        def call():
            # the registration loop's call: forces only (bhtree.bh_forces with
            # count_visits=False, dynamics.py:39); the interaction count of
            # the call comes back as one integer (fga_last_interactions)
            N.check(L.fga_tree_forces(c.handle, N.ptr(q), N.ptr(qm), mm, float(args.theta),
                                      float(p.G), float(p.epsilon) ** 2, N.PREC_FP32, N.ptr(f),
                                      N.ptr(vis) if with_visits else None, None))
            N.check(L.fga_last_interactions(c.handle, ctypes.byref(total)))

        # two untimed calls: the first over a new query count records the
        # warps' traces (one-wave calls then run as split passes)
        for _ in range(2):
            call()
        if sync:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            call()
        return time.perf_counter() - t0, q, qm, f, vis

    lo, hi = m * rank // world, m * (rank + 1) // world
    wall, q, qm, f, vis = slice_calls(lo, hi, world > 1)
    inter_call = float(total.value)
    extra = {}
    # the kernel-level contract (bh_forces_kernel returns forces AND visits):
    # the same calls with the per-query visit counts copied back as well
    wv, q, qm, f, vis = slice_calls(lo, hi, world > 1, with_visits=True)
    if world > 1:
        tv = torch.tensor([wv], dtype=torch.float64, device=torch.device("cuda", local_rank))
        dist.all_reduce(tv, op=dist.ReduceOp.MAX)
        wv = float(tv.item())
    extra["with_visits"] = {
        "value": None,  # (below: all ranks' interactions / the max wall)
        "ms_per_step": 1e3 * wv / args.steps,
        "d2h_bytes_per_step": int(f.nbytes + vis.nbytes + 8) * world,
        "api": "fga_tree_forces with the visits array (the _kernels.bh_forces_kernel contract)"}
    if world == 1 and not args.no_small_m:
        # one rank's slice of an 8-GPU run (rank 3: queries 375k..500k of
        # the template), the same call on this GPU
        w8, *_ = slice_calls(3 * m // 8, 4 * m // 8, False)
        extra["rank_slice_8"] = {
            "queries": 4 * m // 8 - 3 * m // 8, "ms_per_call": 1e3 * w8 / args.steps,
            "interactions_per_s": float(total.value) * args.steps / w8,
            "note": "rank 3's slice of an 8-way run (template rows m*3/8..m*4/8), "
                    "fga_tree_forces from pinned host buffers, wall clock; a one-wave call: "
                    "split passes from the previous call's trace (forces.cu k_bh_op_split)"}
    t = torch.tensor([wall, inter_call], dtype=torch.float64,
                     device=torch.device("cuda", local_rank))
    if world > 1:
        tmax = t[:1].clone()
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        tsum = t[1:].clone()
        dist.all_reduce(tsum)
        wall, inter = float(tmax.item()), float(tsum.item())
    else:
        inter = float(t[1].item())
    extra["with_visits"]["value"] = inter * args.steps / wv
    return {"value": inter * args.steps / wall, "unit": UNIT,
            "h2d_bytes_per_step": int(q.nbytes + qm.nbytes) * world,
            "d2h_bytes_per_step": int(f.nbytes + 8) * world,
            "ms_per_step": 1e3 * wall / args.steps,
            "api": "fga_tree_forces as the registration loop calls the operator (forces out: "
                   "bhtree.bh_forces(count_visits=False), dynamics.py:39; + "
                   "fga_last_interactions for the count), pinned host buffers, initial "
                   "template state, FP32 traversal, wall clock per rank, max over ranks; "
                   "with_visits: the same with the per-query visits copied back",
            "visits_per_query": float(vis.mean()), **extra}


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
        prof = _profile("build").get(str(n)) or {}
        traffic = prof.get("dram_bytes")
        out[str(n)] = {"ms": t * 1e3, "nodes": int(nn.value), "points_per_s": n / t,
                       "roofline": {"bound": "hbm", "unit": "GB/s", "achieved": ach,
                                    "peak": hbm, "frac": ach / hbm,
                                    "peak_source": f"{peak_src} MEASURED_PEAKS.json hbm_gbs",
                                    "work": f"SURVEY §8(d): {BUILD_BYTES_PER_POINT} B/point",
                                    "traffic": traffic,
                                    # the DRAM bytes the build actually moves
                                    # (ncu, all its kernels) over this live time
                                    "dram_frac": (traffic / t / 1e9 / hbm) if traffic else None}}
        del pts, ms, flush
    c.close()
    out["api"] = "fga_tree_build_dev (blob points, unit masses, max_depth 20), median of reps, L2 flushed"
    return out


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
                         "work": "20 FLOP/pair", "traffic": _profile("direct").get("dram_bytes")}}


def run_batched(args, rank, world):
    """configs[4]: the pairs sharded over the ranks with no collective on the
    data path (distributed.register_batch_sharded, every rank one persistent
    kernel over its share), default params (theta 0.6).  `wall_s`: the public
    API from host PointClouds (H2D of the rank's clouds, kernel, D2H of its
    results; gather=False), max over ranks; `kernel_s`: CUDA events around
    fga_register_batch_dev on the same device-resident clouds, max over
    ranks."""
    import ctypes

    import torch

    import paper_2009_14005_b200 as fga
    from paper_2009_14005_b200 import _native as N
    from paper_2009_14005_b200 import synth
    from paper_2009_14005_b200.distributed import register_batch_sharded, shard_of
    dist = None
    if world > 1:
        import torch.distributed as dist
    P = args.batch_pairs
    mine = shard_of(P, rank, world)
    pairs = {p: synth.fragment_pair(p) for p in mine}
    params = fga.default_params()
    register_batch_sharded(lambda p: pairs[p], params=params, n_pairs=P, gather=False)  # warm
    if dist:
        dist.barrier()
    t0 = time.perf_counter()
    br = register_batch_sharded(lambda p: pairs[p], params=params, n_pairs=P, gather=False)
    wall = time.perf_counter() - t0
    its = np.array([br.results[p].iterations for p in mine if br.results[p] is not None])
    inter = float(sum(int(br.interactions[p]) for p in mine))
    failed = int(sum(br.status[p] != 0 for p in mine))
    # the kernel alone on device-resident clouds
    local = [pairs[p] for p in mine]
    xoff = np.zeros(len(local) + 1, np.int64)
    yoff = np.zeros(len(local) + 1, np.int64)
    xoff[1:] = np.cumsum([len(x) for x, _ in local])
    yoff[1:] = np.cumsum([len(y) for _, y in local])
    dev = torch.device("cuda", torch.cuda.current_device())
    Xd = torch.from_numpy(np.concatenate([x.points for x, _ in local])).to(dev)
    Yd = torch.from_numpy(np.concatenate([y.points for _, y in local])).to(dev)
    xo = torch.from_numpy(xoff).to(dev)
    yo = torch.from_numpy(yoff).to(dev)
    res_d = torch.empty(len(local) * ctypes.sizeof(N.CPairResult), dtype=torch.uint8, device=dev)
    cp = N.make_params(params)
    co = fga.registration._c_options(fga.RegisterOptions(), None, None)
    c = N.context(dev.index)
    c.set_stream(torch.cuda.current_stream().cuda_stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    e0.record()
    N.check(N.lib().fga_register_batch_dev(c.handle, Xd.data_ptr(), xo.data_ptr(), Yd.data_ptr(),
                                           yo.data_ptr(), len(local), int(np.diff(xoff).max()),
                                           int(np.diff(yoff).max()), 3, ctypes.byref(cp),
                                           ctypes.byref(co), res_d.data_ptr(), None))
    e1.record()
    torch.cuda.synchronize()
    kernel_s = e0.elapsed_time(e1) / 1e3
    c.set_stream(None)
    if dist:
        t = torch.tensor([wall, kernel_s], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        wall, kernel_s = float(t[0]), float(t[1])
        s2 = torch.tensor([inter, float(failed)], dtype=torch.float64, device=dev)
        dist.all_reduce(s2)
        inter, failed = float(s2[0]), int(s2[1])
        if rank != 0:
            return None
    return {"workload": f"configs[4]: {P} pairs x 4096 pts (synth.fragment_pair: blob/box, "
                        "seeds 100000+p, <=60 deg), default params (theta 0.6)",
            "pairs_per_s": P / kernel_s, "kernel_s": kernel_s,
            "e2e_pairs_per_s": P / wall, "wall_s": wall,
            "interactions_per_s": inter / kernel_s,
            "iterations_min_median_max_rank0": [int(its.min()), float(np.median(its)),
                                                 int(its.max())],
            "failed": failed,
            "api": "distributed.register_batch_sharded (host clouds, wall clock, max over "
                   "ranks) / fga_register_batch_dev (device clouds, CUDA events)",
            "sharding": f"pairs p = rank, rank+{world}, ... over {world} GPU(s), no collective"}


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
    fga.register(x, y, params=p)  # warm (allocations at this size)
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


def run_registration(args, x, y, cpu):
    """Full register() on configs[2] from host numpy (normalize, NIV masses,
    tree, 2x O(NM) energy, the iteration loop, denormalize), median of 3
    after a full-size warm-up; beside it the CPU reference's wall time for
    the same registration, EXTRAPOLATED from the oracle's measured pieces on
    this host (build timed in full; one iteration and one energy from timed
    samples, scaled linearly in M; x the GPU's iteration count)."""
    import paper_2009_14005_b200 as fga
    p = bench_params(args)
    fga.register(x, y, params=p)
    walls = []
    for _ in range(3):
        t0 = time.perf_counter()
        r = fga.register(x, y, params=p)
        walls.append(time.perf_counter() - t0)
    wall = float(np.median(walls))
    out = {"wall_s": wall, "walls_s": walls, "iterations": r.iterations,
           "converged": r.converged, "interactions": int(r.interactions.sum()),
           "timings_ms": r.timings_ms,
           "params": {"theta": p.theta, "G": p.G, "max_iters": p.max_iters,
                      "conv_tol": p.conv_tol},
           "api": "register(x, y) from host numpy, median of 3 calls after a full-size warm-up"}
    if cpu:
        it_s = cpu["iteration_s_extrapolated"]
        gpe_s = cpu["gpe_s_extrapolated"]
        est = cpu["tree_build_s"] + r.iterations * it_s + 2 * gpe_s
        out["cpu_reference_extrapolated"] = {
            "wall_s": est, "cores": cpu["cores"], "kind": "port",
            "parts": {"tree_build_s (measured, 1 core)": cpu["tree_build_s"],
                      "iteration_s (sampled x M/sample)": it_s,
                      "gpe_s (sampled x M/sample)": gpe_s, "iterations": r.iterations},
            "speedup": est / wall, "label": "extrapolated"}
    return out


def run_configs0():
    """configs[0] (the reference's CPU-runnable case): 2,000 x 2,000 blob
    pairs, seeds 0..19 (synth.blob, <= 60 deg / 0.1), theta 0.5, NIV masses.
    GPU register() median wall over the 20 seeds vs the oracle's register()
    (the reference's algorithm) on 1 host core and on all host cores,
    MEASURED; same iteration counts required."""
    import paper_2009_14005_b200 as fga
    from oracle import oracle as orc
    from paper_2009_14005_b200 import synth
    orc.build_lib()
    pairs = []
    for s in range(20):
        rng = synth.rng_from_seed(s)
        x = synth.blob(2000, rng)
        pairs.append((x, synth.misalign(x, synth.random_rigid(rng, np.deg2rad(60), 0.1))))
    p = fga.default_params().replace(theta=0.5)
    fga.register(*pairs[0], params=p)
    gw, its = [], []
    for x, y in pairs:
        t0 = time.perf_counter()
        r = fga.register(x, y, params=p)
        gw.append(time.perf_counter() - t0)
        its.append(r.iterations)
    threads = host_threads()
    cw1, cwn, oits = [], [], []
    for x, y in pairs:
        t0 = time.perf_counter()
        o = orc.register(x.points, y.points, theta=0.5, nthreads=1)
        cw1.append(time.perf_counter() - t0)
        oits.append(o.iterations)
        t0 = time.perf_counter()
        orc.register(x.points, y.points, theta=0.5, nthreads=threads)
        cwn.append(time.perf_counter() - t0)
    return {"workload": "configs[0]: 20 blob pairs 2,000 x 2,000 (seeds 0-19), theta 0.5",
            "gpu_wall_median_s": float(np.median(gw)),
            "cpu_1core_wall_median_s": float(np.median(cw1)),
            "cpu_all_cores_wall_median_s": float(np.median(cwn)), "cpu_cores": threads,
            "speedup_vs_1core": float(np.median(cw1) / np.median(gw)),
            "speedup_vs_all_cores": float(np.median(cwn) / np.median(gw)),
            "iterations_equal": its == oits, "iterations_median": float(np.median(its)),
            "cpu_kind": "port (oracle.register: C tree/forces/energy + numpy Kabsch, "
                        "restating registration.py:91-166)"}


# --------------------------------------------------------------------------- CPU
def cpu_baseline(args, x, y, sample):
    """The C oracle (OpenMP, all host threads) on a bounded sample of the same
    workload and state: tree over the normalized reference (timed, 1 core),
    bh_forces for `sample` template queries at the initial state, and the
    O(NM) energy for 4,096 template points (for the registration
    extrapolation)."""
    from oracle import oracle as orc
    orc.build_lib()
    bp = bench_params(args)
    xn, yn, mx, my, _ = orc.setup(x.points, y.points)
    t0 = time.perf_counter()
    tree = orc.tree_build(xn, mx, 20)
    build_s = time.perf_counter() - t0
    idx = np.random.default_rng(0).choice(len(yn), size=min(sample, len(yn)), replace=False)
    threads = host_threads()
    t0 = time.perf_counter()
    _, visits, acc = orc.bh_forces(tree, yn[idx], my[idx], args.theta, bp.G, bp.epsilon, threads)
    dt = time.perf_counter() - t0
    # the reference as shipped is single-threaded -- one core
    # on a quarter of the sample
    idx1 = idx[: max(1, len(idx) // 4)]
    t0 = time.perf_counter()
    _, _, acc1 = orc.bh_forces(tree, yn[idx1], my[idx1], args.theta, bp.G, bp.epsilon, 1)
    dt1 = time.perf_counter() - t0
    gidx = idx[:4096]
    t0 = time.perf_counter()
    orc.gpe(yn[gidx], my[gidx], xn, mx, bp.G, bp.epsilon, threads)
    gpe_dt = time.perf_counter() - t0
    return {"value": float(acc.sum()) / dt, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"{len(idx)} template queries of the {len(yn)}-point workload at the "
                      f"initial state (oracle bh_forces, theta={args.theta}); tree build "
                      f"{build_s:.2f} s single-threaded",
            "seconds": dt, "visits_per_query": float(visits.mean()),
            "tree_build_s": build_s,
            "iteration_s_extrapolated": dt * len(yn) / len(idx),
            "gpe_s_extrapolated": gpe_dt * len(yn) / len(gidx),
            "one_core": {"value": float(acc1.sum()) / dt1, "unit": UNIT, "cores": 1,
                         "sample": f"{len(idx1)} of the same queries", "seconds": dt1}}


def run_reference(args, rank):
    """--impl reference: the reference's CPU algorithm (C oracle port, all host
    threads) on the same config and state; each step = bh_forces on 16,384
    template queries sampled from the initial state."""
    if rank != 0:
        return None
    from oracle import oracle as orc
    orc.build_lib()
    x, y = workload(args.n, args.seed)
    bp = bench_params(args)
    xn, yn, mx, my, _ = orc.setup(x.points, y.points)
    tree = orc.tree_build(xn, mx, 20)
    threads = host_threads()
    sample = min(16384, len(yn))
    rng = np.random.default_rng(1)

    def step():
        idx = rng.choice(len(yn), size=sample, replace=False)
        t0 = time.perf_counter()
        _, _, acc = orc.bh_forces(tree, yn[idx], my[idx], args.theta, bp.G, bp.epsilon, threads)
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
            "config": config_dict(args, len(x), len(y), tree.node_count, args.gpus),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                             "sample": desc},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}


def main():
    args = parse()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(relaunch(args))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.dry_run:
        line = run_dry(args, rank, world)
        if line is not None:
            print(json.dumps(line), flush=True)
        return
    if args.impl == "reference":
        line = run_reference(args, rank)
        if line is not None:
            print(json.dumps(line), flush=True)
        return
    # FGA_BENCH_FUNCTIONAL=1: a functional check of the N-rank code path on a
    # one-GPU box -- every rank on cuda:0, gloo collectives; its numbers are
    # not measurements (the ranks share one GPU)
    functional = os.environ.get("FGA_BENCH_FUNCTIONAL") == "1"
    if functional:
        local_rank = 0
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        if functional:
            dist.init_process_group("gloo")
        else:
            # NCCL init logging: the communicator's rank count and transport
            # are in the log (stderr), so an N-rank run is verifiable
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    line = run_ours(args, rank, world, local_rank)
    if line is not None and functional:
        line["functional_check_only"] = "all ranks on one GPU (FGA_BENCH_FUNCTIONAL=1)"
    if line is not None:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
