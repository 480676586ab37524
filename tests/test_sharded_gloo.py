"""Template-sharded registration over torch.distributed gloo,
world_size 2, on CPU: the real collective schedule
(paper_2009_14005_b200.distributed.run_sharded) driving a numpy restatement
of the per-shard device session (tests/sharded_backend.py).

Checks: both ranks agree bit for bit; the sharded trajectory equals the
unsharded one to rounding (sums of shard moments == moments of the whole);
and both match the oracle's reference-order registration."""

import os
import socket
import sys

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _case():
    from paper_2009_14005_b200 import synth
    rng = synth.rng_from_seed(5)
    x = synth.blob(1200, rng)
    y = synth.misalign(x, synth.random_rigid(rng, np.deg2rad(40), 0.1))
    return x.points, y.points


def _worker(rank, world, port, outdir):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2009_14005_b200 as fga
    from paper_2009_14005_b200.distributed import run_sharded
    from sharded_backend import NumpyShardBackend
    x, y = _case()
    p = fga.default_params().replace(theta=0.5)
    be = NumpyShardBackend(x, y, p, rank, world)
    res = run_sharded(be, p, fga.RegisterOptions(poll_every=3))
    np.savez(os.path.join(outdir, f"r{rank}.npz"), traj=res["traj"], deltas=res["deltas"],
             it=res["iterations"], gi=res["gpe_initial"], gf=res["gpe_final"])
    dist.destroy_process_group()


def _run(world, tmp_path):
    os.makedirs(tmp_path, exist_ok=True)
    port = _free_port()
    mp.spawn(_worker, args=(world, port, str(tmp_path)), nprocs=world, join=True)
    return [np.load(os.path.join(tmp_path, f"r{r}.npz")) for r in range(world)]


@pytest.mark.timeout(600)
def test_sharded_world2_matches_unsharded_and_oracle(tmp_path, orc):
    one = _run(1, tmp_path / "w1")
    two = _run(2, tmp_path / "w2")
    a, b = two
    assert np.array_equal(a["traj"], b["traj"]) and int(a["it"]) == int(b["it"])
    assert a["gi"] == b["gi"] and a["gf"] == b["gf"]
    ref = one[0]
    assert int(a["it"]) == int(ref["it"])
    assert np.abs(a["traj"] - ref["traj"]).max() < 1e-12
    assert abs(a["gi"] - ref["gi"]) <= 1e-12 * abs(ref["gi"])
    x, y = _case()
    o = orc.register(x, y, theta=0.5)
    assert o.iterations == int(a["it"])
    assert np.abs(np.array(o.trajectory) - a["traj"]).max() < 1e-11
    assert abs(o.gpe_initial - float(a["gi"])) <= 1e-12 * abs(o.gpe_initial)
    assert abs(o.gpe_final - float(a["gf"])) <= 1e-12 * abs(o.gpe_final)
