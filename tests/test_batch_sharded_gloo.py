"""distributed.register_batch_sharded (BASELINE configs[4]: pairs sharded
across GPUs, no collective on the data path) over torch.distributed gloo,
world_size 2, on CPU.  The per-rank batch runner is the oracle's register()
per pair (the device kernel needs a GPU), injected through _register_batch;
what is tested is the package's split (p = rank, rank + world, ...), the lazy
per-rank pair generation and the gather back into pair order, against a
world-1 run and the oracle directly."""

import os
import sys

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
N_PAIRS = 7


def _pair(p):
    from paper_2009_14005_b200 import synth
    return synth.fragment_pair(p, n=400)


def _oracle_batch(pairs, params=None, options=None):
    from oracle import oracle as orc
    from paper_2009_14005_b200.registration import BatchResult
    res = []
    for x, y in pairs:
        o = orc.register(x.points, y.points, theta=params.theta)
        res.append((o.R_orig, o.t_orig, o.iterations, float(x.points[0, 0])))
    return BatchResult(res, [None] * len(res), np.array([len(x) for x, _ in pairs]),
                       np.zeros(len(res), np.int32))


def _worker(rank, world, port, outdir):
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2009_14005_b200 as fga
    from paper_2009_14005_b200.distributed import register_batch_sharded
    made = []

    def lazy(p):
        made.append(p)
        return _pair(p)

    p = fga.default_params()
    br = register_batch_sharded(lazy, params=p, n_pairs=N_PAIRS, _register_batch=_oracle_batch)
    np.savez(os.path.join(outdir, f"r{rank}.npz"),
             R=np.array([r[0] for r in br.results]), t=np.array([r[1] for r in br.results]),
             it=np.array([r[2] for r in br.results]), x0=np.array([r[3] for r in br.results]),
             made=np.array(made), idx=np.array(br.indices), inter=br.interactions)
    dist.destroy_process_group()


def _run(world, tmp_path):
    from test_sharded_gloo import _free_port
    os.makedirs(tmp_path, exist_ok=True)
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    return [np.load(os.path.join(tmp_path, f"r{r}.npz")) for r in range(world)]


@pytest.mark.timeout(600)
def test_batch_sharded_world2_split_and_gather(tmp_path, orc):
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    one = _run(1, tmp_path / "w1")[0]
    a, b = _run(2, tmp_path / "w2")
    # each rank generated and ran only its round-robin share
    assert list(a["made"]) == [0, 2, 4, 6] and list(b["made"]) == [1, 3, 5]
    assert list(a["idx"]) == [0, 2, 4, 6] and list(b["idx"]) == [1, 3, 5]
    # every rank holds the full batch, in pair order, equal to world 1
    for r in (a, b):
        for k in ("R", "t", "it", "x0", "inter"):
            assert np.array_equal(r[k], one[k]), k
    # and pair p is pair p
    for p in (0, 3, 6):
        x, y = _pair(p)
        o = orc.register(x.points, y.points, theta=0.6)
        assert np.array_equal(a["R"][p], o.R_orig) and int(a["it"][p]) == o.iterations
        assert a["x0"][p] == x.points[0, 0]
