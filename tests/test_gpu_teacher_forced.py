"""Teacher-forced iteration parity (SURVEY §8(c) protocol 2): the session is
put into the reference's exact state entering iteration k (positions,
velocities, [R_acc | t_acc], from the golden run of register() on config-1
seed 0, tests/golden/make_golden.py) and runs ONE iteration; its
[R_acc | t_acc] and the state it hands to iteration k+1 must equal the
reference's (registration.py:130-154).  The same golden states pin the
force operator on the session's tree (bhtree.bh_forces, bhtree.py:125-152).
GPU only."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fga():
    import paper_2009_14005_b200 as f
    return f


def _session(fga, g, precision):
    from paper_2009_14005_b200.engine import Session
    x, y = fga.PointCloud(g["s0/x"]), fga.PointCloud(g["s0/y"])
    p = fga.default_params().replace(theta=0.5)
    return Session(x, y, p, fga.RegisterOptions(compute_gpe=False, record_iterations=True,
                                                precision=precision))


def test_session_setup_state_matches_reference(golden, fga):
    g = golden("register")
    s = _session(fga, g, "fp64")
    st = s.get_state()
    mx, my = s.masses()
    s.finish()
    assert st["iteration"] == 0
    assert np.array_equal(st["positions"], g["tf/yn"])  # normalized template, bit-exact
    assert not st["velocities"].any()
    assert np.array_equal(mx, g["tf/mass_x"]) and np.array_equal(my, g["tf/mass_y"])
    assert np.array_equal(st["R_acc"], np.eye(3)) and not st["t_acc"].any()


@pytest.mark.parametrize("it", [0, 1, 3])
@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_teacher_forced_iteration(golden, fga, it, precision):
    g = golden("register")
    s = _session(fga, g, precision)
    prev = g[f"tf/it{it}/traj_prev"]
    s.set_state(g[f"tf/it{it}/pos"], g[f"tf/it{it}/vel"], prev[:, :3], prev[:, 3], it)
    s.iterate(1)
    st = s.get_state()
    res = s.finish()
    assert res.iterations == it + 1
    tol = 2e-6 if precision == "fp32" else 1e-11
    assert np.abs(res.trajectory[it] - g[f"tf/it{it}/traj"]).max() < tol
    if it == 0:  # the state entering iteration 1
        assert np.abs(st["positions"] - g["tf/it1/pos"]).max() < tol
        assert np.abs(st["velocities"] - g["tf/it1/vel"]).max() < tol * 10


@pytest.mark.parametrize("it", [0, 1, 3])
def test_teacher_forced_forces_on_session_tree(golden, fga, it):
    """bh_forces on the GPU-built tree of the normalized reference cloud at
    the reference's own iteration-k template state.  The GPU tree's topology
    is the reference's bit for bit, its centres of mass agree to ~1e-15
    relative (children-first summation vs the reference's per-node sums), so
    the fp64 forces agree to 1e-11 of the largest force (bit-exact on the
    reference's own tree: test_bh_forces_fp64_bit_exact_on_reference_tree)."""
    from paper_2009_14005_b200 import bhtree
    g = golden("register")
    p = fga.default_params().replace(theta=0.5)
    t = bhtree.build(fga.PointCloud(g["tf/xn"]), g["tf/mass_x"], p.max_depth)
    f, v = bhtree.bh_forces(t, g[f"tf/it{it}/pos"], g["tf/mass_y"], p, count_visits=True,
                            precision="fp64")
    scale = np.linalg.norm(g[f"tf/it{it}/grav"], axis=1).max()
    assert np.abs(f - g[f"tf/it{it}/grav"]).max() <= 1e-11 * scale
    f32 = bhtree.bh_forces(t, g[f"tf/it{it}/pos"], g["tf/mass_y"], p, precision="fp32")
    assert np.abs(f32 - g[f"tf/it{it}/grav"]).max() <= 1e-5 * scale


def test_checkpoint_resume_is_exact(fga):
    """get_state after k iterations, set_state into a fresh session, continue:
    the same trajectory as an uninterrupted run (fp64)."""
    from paper_2009_14005_b200 import synth
    from paper_2009_14005_b200.engine import Session
    rng = synth.rng_from_seed(11)
    x = synth.blob(3000, rng)
    y = synth.misalign(x, synth.random_rigid(rng, np.deg2rad(40), 0.1))
    p = fga.default_params().replace(theta=0.5, conv_tol=1e-300, max_iters=8)
    o = fga.RegisterOptions(compute_gpe=False, record_iterations=True, precision="fp64")
    a = Session(x, y, p, o)
    a.iterate(8)
    ra = a.finish()
    b = Session(x, y, p, o)
    b.iterate(3)
    ck = b.get_state()
    b.finish()
    c = Session(x, y, p, o)
    c.set_state(ck["positions"], ck["velocities"], ck["R_acc"], ck["t_acc"], ck["iteration"])
    c.iterate(5)
    rc = c.finish()
    assert rc.iterations == 8
    assert np.abs(rc.trajectory[3:] - ra.trajectory[3:]).max() < 1e-10


@pytest.mark.parametrize("case", ["c2", "c4"])
@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_teacher_forced_config_shapes(golden, fga, case, precision):
    """configs[1]/[3]-shaped pairs (6k-point LiDAR street scan; 40%-overlap
    pair with outliers and inhomogeneous density): the session's mass fields
    are the reference's bit for bit, and from the reference's own states one
    GPU iteration reproduces its [R_acc | t_acc] (tests/golden/tf_configs.npz)."""
    from paper_2009_14005_b200.engine import Session
    g = golden("tf_configs")
    k = case + "/"
    p = fga.default_params().replace(theta=0.5, G=float(g[k + "G"]), max_iters=3,
                                     conv_tol=1e-300)
    o = fga.RegisterOptions(compute_gpe=False, record_iterations=True, precision=precision)
    tol = 2e-5 if precision == "fp32" else 1e-10
    s = Session(fga.PointCloud(g[k + "x"]), fga.PointCloud(g[k + "y"]), p, o)
    mx, my = s.masses()
    assert np.array_equal(mx, g[k + "mass_x"]) and np.array_equal(my, g[k + "mass_y"])
    s.iterate(1)  # iteration 0 from the session's own setup
    st = s.get_state()
    r0 = s.finish()
    assert np.abs(r0.trajectory[0] - g[k + "traj"][0]).max() < tol
    scale = np.abs(g[k + "pos"][0]).max()
    assert np.abs(st["positions"] - g[k + "pos"][0]).max() < tol * max(scale, 1.0)
    for it in (1, 2):
        s = Session(fga.PointCloud(g[k + "x"]), fga.PointCloud(g[k + "y"]), p, o)
        prev = g[k + "traj"][it - 1]
        s.set_state(g[k + "pos"][it - 1], g[k + "vel"][it - 1], prev[:, :3], prev[:, 3], it)
        s.iterate(1)
        r = s.finish()
        assert np.abs(r.trajectory[it] - g[k + "traj"][it]).max() < tol


def test_device_checkpoint_restore_is_exact(fga):
    """fga_session_checkpoint: save on the device after k iterations, run on,
    restore, run the same iterations again -- bitwise the same transforms
    (bench.py re-times the initial state this way)."""
    from paper_2009_14005_b200 import synth
    from paper_2009_14005_b200.engine import Session
    rng = synth.rng_from_seed(12)
    x = synth.blob(5000, rng)
    y = synth.misalign(x, synth.random_rigid(rng, np.deg2rad(40), 0.1))
    p = fga.default_params().replace(theta=0.5, conv_tol=1e-300, max_iters=20)
    s = Session(x, y, p, fga.RegisterOptions(compute_gpe=False, record_iterations=True))
    s.iterate(3)
    s.checkpoint()
    s.iterate(2)
    a = s.get_state()
    s.restore()
    s.iterate(2)
    b = s.get_state()
    s.finish()
    assert a["iteration"] == b["iteration"] == 5
    assert np.array_equal(a["positions"], b["positions"])
    assert np.array_equal(a["velocities"], b["velocities"])
    assert np.array_equal(a["R_acc"], b["R_acc"]) and np.array_equal(a["t_acc"], b["t_acc"])
