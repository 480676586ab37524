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
