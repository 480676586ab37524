"""Repeat-run determinism of the kernels with shared-memory / atomic
cooperation (the race-prone code VERDICT r01 asked a sanitizer for;
compute-sanitizer is closed on this GPU pool): every value is designed to be
a fixed function of the input (fixed-order sums, slot-ordered child folds,
dynamic work claiming only over independent units), so a data race would
show up as run-to-run differences.  Each case is rerun many times and must
be bitwise identical.  The same suite also runs against the FGA_CHECKS=1
build (device-side bounds / arrival-counter asserts, tools/check_build.sh).
GPU only."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _cases():
    rng = np.random.default_rng(21)
    pts = {
        "n129": rng.uniform(-2, 3, size=(129, 3)),
        "n4097": rng.uniform(-2, 3, size=(4097, 3)),
        "dup_runs": np.repeat(rng.uniform(-1, 1, size=(5, 3)), 300, axis=0)[rng.permutation(1500)],
        "tight_cluster": np.vstack([rng.uniform(-1, 1, size=(700, 3)),
                                    0.3 + rng.normal(size=(700, 3)) * 1e-9]),
    }
    from paper_2009_14005_b200 import synth
    pts["blob200k"] = synth.blob(200_000, synth.rng_from_seed(22)).points * 5
    return pts


@pytest.mark.parametrize("name", ["n129", "n4097", "dup_runs", "tight_cluster", "blob200k"])
def test_tree_build_repeats_bitwise(name):
    import paper_2009_14005_b200 as fga
    from paper_2009_14005_b200 import bhtree
    p = _cases()[name]
    m = np.random.default_rng(5).uniform(0.001, 0.02, size=len(p))
    ref = bhtree.build(fga.PointCloud(p), m, 20)
    for _ in range(20 if len(p) < 10000 else 6):
        t = bhtree.build(fga.PointCloud(p), m, 20)
        for k in ("children", "com", "mass", "length", "occupancy", "depth", "bbox_min",
                  "bbox_max"):
            assert np.array_equal(getattr(t, k), getattr(ref, k)), k


def test_batched_kernel_repeats_bitwise():
    import paper_2009_14005_b200 as fga
    from paper_2009_14005_b200 import synth
    pairs = [synth.fragment_pair(p, n=1500 + 300 * (p % 5)) for p in range(24)]
    p = fga.default_params()
    first = fga.register_batch(pairs, params=p)
    for _ in range(4):
        again = fga.register_batch(pairs, params=p)
        assert np.array_equal(again.interactions, first.interactions)
        for a, b in zip(again.results, first.results):
            assert a.iterations == b.iterations
            assert np.array_equal(a.transform.rotation, b.transform.rotation)
            assert np.array_equal(a.transform.translation, b.transform.translation)
            assert a.gpe_initial == b.gpe_initial and a.gpe_final == b.gpe_final


def test_register_and_forces_repeat_bitwise():
    import paper_2009_14005_b200 as fga
    from paper_2009_14005_b200 import bhtree, synth
    x, y, _ = synth.configs1_pair(60_000)
    p = fga.default_params().replace(theta=0.5, G=0.2)
    o = fga.RegisterOptions(record_iterations=True)
    r0 = fga.register(x, y, params=p, options=o)
    for _ in range(3):
        r = fga.register(x, y, params=p, options=o)
        assert r.iterations == r0.iterations
        assert np.array_equal(r.trajectory, r0.trajectory)
        assert r.gpe_initial == r0.gpe_initial and r.gpe_final == r0.gpe_final
    xn, yn, _ = fga.normalize_pair(x, y, -5.0, 5.0)
    t = bhtree.build(xn, np.full(len(xn), 1e-3), 20)
    f0, v0 = bhtree.bh_forces(t, yn.points, 0.05, p, count_visits=True, precision="fp32")
    for _ in range(4):
        f, v = bhtree.bh_forces(t, yn.points, 0.05, p, count_visits=True, precision="fp32")
        assert np.array_equal(f, f0) and np.array_equal(v, v0)
