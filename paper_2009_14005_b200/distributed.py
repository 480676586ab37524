"""Multi-GPU registration of one large pair by template sharding.

One process per GPU (torchrun).  Every rank receives the FULL clouds, runs the
identical device setup (normalization, masses, tree -- deterministic, so the
replicated tree is bit-identical everywhere) and owns a contiguous chunk of
the Hilbert-ordered template.  Per iteration the only exchange is ONE
all-reduce (sum) of the 18-double sums buffer: the shifted Kabsch moments
(sum u, sum w, sum w u^T = 15 doubles, the covariance and centroid partials
of procrustes.py:20-25), the interaction/visit counters and, when tracing,
the energy partial.  Every rank then runs the same fp64 SVD update, so the
transforms (and the stop decision) agree on all ranks without further
traffic.  torch.distributed supplies the collective (NCCL over NVLink on
B200; gloo in the CPU tests, where a test backend stands in for libfga).

The driver is written against a small backend protocol so the host logic --
the collective schedule and the stop/poll protocol -- is testable on CPU.
"""

from __future__ import annotations

import torch
import torch.distributed as dist

from .core import FgaParams, default_params
from .engine import SUMS_LEN, Session
from .registration import RegisterOptions


class _LibBackend:
    """libfga session bound to a torch tensor as its sums buffer."""

    def __init__(self, x, y, params, options, rank, world, device):
        torch.cuda.set_device(device)
        self.sums = torch.zeros(SUMS_LEN, dtype=torch.float64, device=f"cuda:{device}")
        stream = torch.cuda.current_stream().cuda_stream
        self.s = Session(x, y, params, options, shard_rank=rank, shard_count=world,
                         device=device, stream=stream)
        self.s.bind_sums(self.sums.data_ptr())

    def forces(self):
        self.s.forces()

    def update(self):
        self.s.update()

    def gpe(self):
        self.s.gpe()

    def take_gpe(self):
        return self.s.take_gpe()

    def set_gpe(self, which, v):
        self.s.set_gpe(which, v)

    def apply_pending(self):
        self.s.apply_pending()

    def poll(self):
        return self.s.poll()

    def finish(self):
        return self.s.finish()


def run_sharded(backend, params: FgaParams, options: RegisterOptions, group=None):
    """The collective schedule shared by the GPU driver and the CPU tests."""
    def allreduce():
        dist.all_reduce(backend.sums, op=dist.ReduceOp.SUM, group=group)

    if options.compute_gpe:
        backend.gpe()
        allreduce()
        backend.set_gpe(0, backend.take_gpe())
    passes = 0
    done = False
    while not done:
        k = max(1, min(int(options.poll_every), params.max_iters - passes))
        for _ in range(k):
            backend.forces()
            allreduce()
            backend.update()
            passes += 1
        done, _ = backend.poll()
        if passes >= params.max_iters:
            done = True
    backend.apply_pending()
    if options.compute_gpe:
        backend.gpe()
        allreduce()
        backend.set_gpe(1, backend.take_gpe())
    return backend.finish()


def register_sharded(x, y, params: FgaParams | None = None,
                     options: RegisterOptions | None = None, group=None, device=None):
    """register() with the template split across the ranks of ``group``;
    returns the same RegistrationResult on every rank."""
    params = params or default_params()
    options = options or RegisterOptions()
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    if device is None:
        device = torch.cuda.current_device()
    backend = _LibBackend(x, y, params, options, rank, world, device)
    return run_sharded(backend, params, options, group)


def shard_of(n_pairs: int, rank: int, world: int) -> list[int]:
    """The pairs rank `rank` of `world` registers: p = rank, rank + world, ...
    (round robin, so fragment pairs of mixed difficulty spread evenly)."""
    return list(range(rank, n_pairs, world))


def register_batch_sharded(pairs, params: FgaParams | None = None,
                           options: RegisterOptions | None = None, group=None,
                           gather: bool = True, n_pairs: int | None = None,
                           _register_batch=None):
    """Many independent pairs (BASELINE configs[4]) sharded across the ranks
    of ``group`` with NO collective on the data path: each rank runs
    register_batch (one persistent kernel) on its own share
    (``shard_of``) and the results are only gathered at the end.

    ``pairs`` is either a sequence of (x, y) PointCloud pairs (every rank may
    pass the full list; only its share is touched) or a callable p -> (x, y)
    with ``n_pairs`` given, so a rank materializes only its own pairs.
    Returns a registration.BatchResult in pair order: with ``gather`` the full
    batch on every rank (dist.all_gather_object of the per-rank results),
    otherwise this rank's entries only (the other slots None) and
    ``.indices`` = the pairs it ran.  Reference unit of work:
    registration.register per pair (registration.py:91-166)."""
    from .registration import BatchResult, register_batch

    rank = dist.get_rank(group) if dist.is_initialized() else 0
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if callable(pairs):
        if n_pairs is None:
            raise ValueError("n_pairs is required when pairs is a callable")
        total = int(n_pairs)
        mine = shard_of(total, rank, world)
        local = [pairs(p) for p in mine]
    else:
        pairs = list(pairs)
        total = len(pairs)
        mine = shard_of(total, rank, world)
        local = [pairs[p] for p in mine]
    run = _register_batch or register_batch
    br = run(local, params=params, options=options)
    out = BatchResult([None] * total, [None] * total, None, None)
    out.indices = mine
    parts = [(mine, br.results, br.errors, None if br.interactions is None else
              list(br.interactions), None if br.status is None else list(br.status))]
    if gather and world > 1:
        allparts = [None] * world
        dist.all_gather_object(allparts, parts[0], group=group)
        parts = allparts
    inter = [0] * total
    status = [0] * total
    for idx, res, err, it, st in parts:
        for k, p in enumerate(idx):
            out.results[p] = res[k]
            out.errors[p] = err[k]
            if it is not None:
                inter[p] = int(it[k])
            if st is not None:
                status[p] = int(st[k])
    import numpy as np
    out.interactions = np.array(inter, np.int64)
    out.status = np.array(status, np.int32)
    return out
