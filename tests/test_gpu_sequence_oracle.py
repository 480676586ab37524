"""register_sequence (registration.py:178-206) against the oracle's
restatement of it (oracle.register_sequence): every pairwise transform, the
failed flags of a degenerate pair (identity + failed, registration.py:197-200)
and the composed poses (core.py:87-96), on each of the device's three paths:
fragment-sized frames (one batched kernel), frames above 8192 points (host
threads, one context per thread) and D = 2 frames.  GPU only.

Tolerances (north_star): R within 1e-4 rad, t within 1e-4 * scene extent,
the same iteration counts as the oracle (checked through the pairwise
transforms: a one-iteration difference moves R, t by ~1e-2)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _rot_err(Ra, Rb):
    d = len(Ra)
    c = np.trace(Ra.T @ Rb) / 2 if d == 2 else (np.trace(Ra.T @ Rb) - 1) / 2
    return float(np.arccos(np.clip(c, -1, 1)))


def _frames(n, k, seed, degenerate_tail=False):
    from paper_2009_14005_b200 import PointCloud, synth
    rng = synth.rng_from_seed(seed)
    frames = [synth.blob(n, rng)]
    for _ in range(k - 1):
        frames.append(synth.misalign(frames[-1], synth.random_rigid(rng, np.deg2rad(8), 0.03)))
    if degenerate_tail:
        # an empty frame (both of its pairs raise EmptyCloud), then two frames
        # whose every point coincides with its centroid (dyadic coordinates,
        # so numpy's mean is exact): that pair raises DegenerateExtent
        # (normalize.py:52-53)
        frames.append(PointCloud(np.zeros((0, 3))))
        frames.append(PointCloud(np.tile([[0.5, -0.25, 0.125]], (n // 2, 1))))
        frames.append(PointCloud(np.tile([[0.25, 0.5, -0.375]], (n // 4, 1))))
    return frames


def _check(seq, ref, frames):
    extent = max(np.ptp(f.points, axis=0).max() for f in frames if len(f))
    assert list(seq.failed) == list(ref.failed)
    assert len(seq.pairwise) == len(ref.pairwise)
    for k, (tf, (R, t)) in enumerate(zip(seq.pairwise, ref.pairwise)):
        assert _rot_err(tf.rotation, R) < 1e-4, k
        assert np.abs(tf.translation - t).max() < 1e-4 * extent, k
        if ref.failed[k]:
            assert np.array_equal(tf.rotation, np.eye(len(t)))
            assert np.array_equal(tf.translation, np.zeros(len(t)))
    for k, (pose, (P, p)) in enumerate(zip(seq.trajectory, ref.trajectory)):
        assert _rot_err(pose.rotation, P) < 1e-4 * max(k, 1), k
        assert np.abs(pose.translation - p).max() < 1e-4 * extent * max(k, 1), k


@pytest.mark.parametrize("n,label", [(1500, "batched"), (9000, "threaded")])
def test_sequence_matches_oracle(orc, n, label):
    import paper_2009_14005_b200 as fga
    frames = _frames(n, 4, 300 + n, degenerate_tail=True)
    seq = fga.register_sequence(frames)
    ref = orc.register_sequence([f.points for f in frames], theta=fga.default_params().theta)
    assert ref.failed == [False, False, False, True, True, True]
    _check(seq, ref, frames)


def test_sequence_two_d_matches_oracle(orc):
    import paper_2009_14005_b200 as fga
    rng = np.random.default_rng(11)
    base = rng.normal(size=(700, 2)) * [1.0, 0.4]
    frames = [fga.PointCloud(base)]
    for k in range(3):
        a = 0.04 * (k + 1)
        R = np.array([[np.cos(a), -np.sin(a)], [np.sin(a), np.cos(a)]])
        frames.append(fga.PointCloud(frames[-1].points @ R.T + [0.01, -0.02]))
    frames.append(fga.PointCloud(np.zeros((0, 2))))
    frames.append(fga.PointCloud(np.tile([[0.5, 0.5]], (64, 1))))
    frames.append(fga.PointCloud(np.tile([[-0.5, 0.25]], (32, 1))))
    seq = fga.register_sequence(frames)
    ref = orc.register_sequence([f.points for f in frames], theta=fga.default_params().theta)
    assert ref.failed == [False, False, False, True, True, True]
    _check(seq, ref, frames)
