"""Template sharding on the device path.  One GPU only: two
shards run as two library sessions in one process, their 18-double sums
buffers combined with a device add -- the all-reduce's arithmetic without
ranks that wait on one another -- then the NCCL driver itself at world 1."""

import os

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _pair(n=3000, seed=21):
    from paper_2009_14005_b200 import synth
    rng = synth.rng_from_seed(seed)
    x = synth.blob(n, rng)
    return x, synth.misalign(x, synth.random_rigid(rng, np.deg2rad(45), 0.1))


def test_two_shards_equal_one(orc):
    import paper_2009_14005_b200 as fga
    from paper_2009_14005_b200 import _native as N
    from paper_2009_14005_b200.engine import Session
    x, y = _pair()
    p = fga.default_params().replace(theta=0.5)
    o = fga.RegisterOptions(compute_gpe=False)
    ref = fga.register(x, y, params=p, options=fga.RegisterOptions(record_iterations=True))
    stream = torch.cuda.current_stream().cuda_stream
    shards = [Session(x, y, p, o, shard_rank=r, shard_count=2, stream=stream,
                      ctx=N.Context(0)) for r in range(2)]
    bufs = [torch.zeros(18, dtype=torch.float64, device="cuda") for _ in shards]
    for s, b in zip(shards, bufs):
        s.bind_sums(b.data_ptr())
    assert sum(s.m_local for s in shards) == len(y)
    done = False
    while not done:
        for s in shards:
            s.forces()
        tot = bufs[0] + bufs[1]
        for b in bufs:
            b.copy_(tot)
        for s in shards:
            s.update()
        done, it = shards[0].poll()
        assert shards[1].poll() == (done, it)
    r0, r1 = shards[0].finish(), shards[1].finish()
    assert np.array_equal(r0.trajectory, r1.trajectory)
    assert r0.iterations == ref.iterations and r0.converged == ref.converged
    assert np.abs(r0.trajectory - ref.trajectory).max() < 1e-10
    assert np.array_equal(r0.interactions, ref.interactions)


def test_register_sharded_nccl_world1():
    import torch.distributed as dist
    import paper_2009_14005_b200 as fga
    from paper_2009_14005_b200.distributed import register_sharded
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29533")
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        x, y = _pair(2000, 22)
        p = fga.default_params().replace(theta=0.5)
        opts = fga.RegisterOptions(record_iterations=True)
        a = register_sharded(x, y, p, opts)
        b = fga.register(x, y, params=p, options=opts)
        assert a.iterations == b.iterations
        assert np.array_equal(a.trajectory, b.trajectory)
        assert a.gpe_initial == b.gpe_initial and a.gpe_final == b.gpe_final
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("count", [2, 3, 8])
def test_cost_balanced_shards_partition_the_template(count):
    """Cost-balanced cuts (capi.cu balanced_cut: sampled visit counts in
    Morton order): the shards' sizes add up to the template, they are not
    the equal-count split on a clustered cloud, their accepted interactions
    add up to the unsharded pass's, and FGA_SHARD_BALANCE is not needed for
    correctness (the per-query forces do not depend on the cut)."""
    import paper_2009_14005_b200 as fga
    from paper_2009_14005_b200 import _native as N
    from paper_2009_14005_b200.engine import SUM_ACCEPTED, Session
    x, y = _pair(n=40000, seed=5)
    p = fga.default_params().replace(theta=0.5, max_iters=1)
    o = fga.RegisterOptions(compute_gpe=False)
    stream = torch.cuda.current_stream().cuda_stream

    def accepted(rank, cnt):
        s = Session(x, y, p, o, shard_rank=rank, shard_count=cnt, stream=stream,
                    ctx=N.Context(0))
        b = torch.zeros(18, dtype=torch.float64, device="cuda")
        s.bind_sums(b.data_ptr())
        s.forces()
        torch.cuda.synchronize()
        a, m = float(b[SUM_ACCEPTED].item()), s.m_local
        s.finish()
        return a, m

    parts = [accepted(r, count) for r in range(count)]
    whole, m_all = accepted(0, 1)
    assert m_all == len(y)
    assert sum(m for _, m in parts) == len(y)
    assert sum(a for a, _ in parts) == whole
    equal = [len(y) * (r + 1) // count - len(y) * r // count for r in range(count)]
    assert [m for _, m in parts] != equal
