"""Seeded synthetic inputs for the benchmark configurations (BASELINE.json).

``blob``, ``random_rigid`` and ``misalign`` draw from a PCG64 generator in the
same order as the reference's generators (gravreg/synth.py:13-14, :55-61,
:102-145), so a seed gives the same clouds the reference's own harness uses.
``lidar_scan`` (config 2) and ``partial_overlap`` (config 4) are new: the
reference ships no LiDAR-shaped or partial-overlap generator.
"""

from __future__ import annotations

import numpy as np

from .core import PointCloud, RigidTransform


def rng_from_seed(seed):
    return np.random.Generator(np.random.PCG64(seed))


def blob(n, rng, k=6):
    """k anisotropic Gaussian clusters in the unit cube (synth.py:55-61)."""
    centres = rng.uniform(-0.5, 0.5, size=(k, 3))
    spreads = rng.uniform(0.10, 0.18, size=(k, 3))
    label = rng.integers(0, k, size=n)
    return PointCloud(centres[label] + rng.normal(size=(n, 3)) * spreads[label])


def bumped_box(n, rng):
    """Cuboid shell [+-0.5, +-0.35, +-0.25] with an off-centre bump on the +x
    face (synth.py:64-84)."""
    half = np.array([0.5, 0.35, 0.25])
    face = rng.integers(0, 6, size=n)
    uv = rng.uniform(-1.0, 1.0, size=(n, 2))
    axis = face % 3
    sign = np.where(face < 3, 1.0, -1.0)
    pts = np.empty((n, 3))
    for k in range(3):
        sel = axis == k
        others = [j for j in range(3) if j != k]
        pts[sel, k] = sign[sel] * half[k]
        pts[sel, others[0]] = uv[sel, 0] * half[others[0]]
        pts[sel, others[1]] = uv[sel, 1] * half[others[1]]
    bump = (np.abs(pts[:, 0] - half[0]) < 1e-9) & (
        np.hypot(pts[:, 1] - 0.15, pts[:, 2] - 0.08) < 0.12)
    pts[bump, 0] += 0.1
    return PointCloud(pts)


def axis_angle(axis, angle):
    """Rodrigues rotation about a unit axis."""
    u = np.asarray(axis, dtype=np.float64)
    u = u / np.linalg.norm(u)
    K = np.array([[0.0, -u[2], u[1]], [u[2], 0.0, -u[0]], [-u[1], u[0], 0.0]])
    return np.eye(3) + np.sin(angle) * K + (1.0 - np.cos(angle)) * (K @ K)


def random_rotation(rng, max_angle_rad):
    angle = rng.uniform(0.0, max_angle_rad)
    axis = rng.normal(size=3)
    return axis_angle(axis / np.linalg.norm(axis), angle)


def euler_rotation(rng, max_angle_rad):
    """Rz(c) Ry(b) Rx(a) with a, b, c ~ U(0, max) (synth.py:109-118)."""
    rx, ry, rz = rng.uniform(0.0, max_angle_rad, size=3)
    return (axis_angle([0.0, 0.0, 1.0], rz) @ axis_angle([0.0, 1.0, 0.0], ry)
            @ axis_angle([1.0, 0.0, 0.0], rx))


def random_rigid(rng, max_angle_rad, max_translation, euler=False):
    """Uniform-axis rotation with angle U(0, max) (or per-axis Euler angles),
    translation of length U(0, max_t) along a uniform direction
    (synth.py:134-139)."""
    R = euler_rotation(rng, max_angle_rad) if euler else random_rotation(rng, max_angle_rad)
    direction = rng.normal(size=3)
    direction /= np.linalg.norm(direction)
    return RigidTransform(R, direction * rng.uniform(0.0, max_translation))


def misalign(cloud: PointCloud, gt: RigidTransform) -> PointCloud:
    """Template y = gt^{-1}(x), so gt maps y back onto x (synth.py:142-145)."""
    return PointCloud(gt.inverse().apply(cloud.points))


def add_uniform_noise(cloud: PointCloud, fraction, rng, low=-0.5, high=0.5):
    """Append fraction*n uniform outliers (synth.py:158-164)."""
    extra = int(round(fraction * len(cloud)))
    if extra == 0:
        return cloud
    return PointCloud(np.vstack([cloud.points, rng.uniform(low, high, size=(extra, cloud.dim))]))


def lidar_scene(rng):
    """The street of lidar_scan: 20 box "cars" (4.5 x 1.8 x 1.5 m) in four
    lanes and 12 poles (0.3 x 0.3 x 6 m) along the facades, as (lo, hi) boxes."""
    boxes = []
    for _ in range(20):
        cx = rng.uniform(-40, 40)
        cy = rng.choice([-5.0, -2.0, 2.0, 5.0]) + rng.uniform(-0.3, 0.3)
        boxes.append(((cx - 2.25, cy - 0.9, 0.0), (cx + 2.25, cy + 0.9, 1.5)))
    for _ in range(12):
        cx = rng.uniform(-40, 40)
        cy = rng.choice([-7.0, 7.0])
        boxes.append(((cx - 0.15, cy - 0.15, 0.0), (cx + 0.15, cy + 0.15, 6.0)))
    return boxes


def lidar_scan(n, rng, sensor_height=1.73, scene=None, pose=None):
    """A spinning 64-beam scan (elevation -24.9..+2 deg, 0.18 deg azimuth
    steps) of a street: ground plane, two facades at +-8 m, 20 box "cars" and
    poles; range noise N(0, 2 cm); subsampled to exactly n returns, so the
    density falls off ~1/r^2 like a real sensor (config 2).

    `scene` (lidar_scene) fixes the street; `pose` (RigidTransform, sensor
    frame -> street frame) moves the sensor: the returns are in the SENSOR's
    frame, so a second scan from `pose` is a realistic next frame whose
    registration onto the first recovers `pose` (different sampling, not a
    rigid copy)."""
    elev = np.deg2rad(np.linspace(-24.9, 2.0, 64))
    az = np.deg2rad(np.arange(0.0, 360.0, 0.18))
    E, A = np.meshgrid(elev, az, indexing="ij")
    d = np.stack([np.cos(E) * np.cos(A), np.cos(E) * np.sin(A), np.sin(E)], -1).reshape(-1, 3)
    o = np.array([0.0, 0.0, sensor_height])
    if pose is not None:  # rays of the moved sensor, in street coordinates
        d = d @ pose.rotation.T
        o = pose.rotation @ o + pose.translation
    t = np.full(len(d), np.inf)
    dz = d[:, 2]
    with np.errstate(divide="ignore", invalid="ignore"):
        # ground z = 0
        t = np.minimum(t, np.where(dz < 0, -o[2] / dz, np.inf))
        # facades y = +-8 (height 0..12 m)
        for wall in (8.0, -8.0):
            tw = np.where(d[:, 1] * np.sign(wall - o[1]) > 0, (wall - o[1]) / d[:, 1], np.inf)
            zw = o[2] + tw * dz
            t = np.minimum(t, np.where((zw >= 0) & (zw <= 12.0), tw, np.inf))
    boxes = scene if scene is not None else lidar_scene(rng)
    with np.errstate(divide="ignore", invalid="ignore"):
        inv = 1.0 / d
        for lo, hi in boxes:
            t1 = (np.array(lo) - o) * inv
            t2 = (np.array(hi) - o) * inv
            tmin = np.nanmax(np.minimum(t1, t2), axis=1)
            tmax = np.nanmin(np.maximum(t1, t2), axis=1)
            hit = (tmax >= np.maximum(tmin, 0)) & (tmin > 0)
            t = np.where(hit & (tmin < t), tmin, t)
    ok = np.isfinite(t) & (t < 80.0)
    r = t[ok] + rng.normal(0.0, 0.02, size=ok.sum())
    pts = o + d[ok] * r[:, None]
    if pose is not None:  # street -> sensor frame
        pts = (pts - pose.translation) @ pose.rotation
    if len(pts) >= n:
        pts = pts[np.sort(rng.choice(len(pts), size=n, replace=False))]
    else:  # densify by jittered resampling to reach exactly n returns
        extra = pts[rng.integers(0, len(pts), size=n - len(pts))]
        pts = np.vstack([pts, extra + rng.normal(0.0, 0.02, size=extra.shape)])
    return PointCloud(pts)


def partial_overlap(n, rng, overlap=0.4, outliers=0.05):
    """Config 4: inhomogeneously thinned blob split into two clouds sharing
    `overlap` of their points, each padded with `outliers` uniform noise."""
    base_n = int(round(n * (1 - outliers) / ((1 + overlap) / 2 + (1 - overlap) / 2) * 1.25 + 1))
    c = blob(base_n * 3, rng).points
    centre = c[rng.integers(0, len(c))]
    keep = rng.uniform(size=len(c)) < 0.2 + 0.8 * np.exp(
        -((c - centre) ** 2).sum(1) / (2 * 0.25**2))
    c = c[keep]
    c = c[np.argsort(c[:, 0])]
    inliers = int(round(n * (1 - outliers)))
    share = int(round(inliers * overlap))
    first = inliers - share
    # x takes [0, inliers), y takes [first, first + inliers) of the x-sorted base
    total = first + inliers
    if len(c) < total:
        c = np.vstack([c, c[rng.integers(0, len(c), size=total - len(c))] +
                       rng.normal(0, 0.005, size=(total - len(c), 3))])
        c = c[np.argsort(c[:, 0])]
    idx = np.sort(rng.choice(len(c), size=total, replace=False))
    c = c[idx]
    x = PointCloud(c[:inliers])
    y = PointCloud(c[first:first + inliers])
    x = add_uniform_noise(x, (n - inliers) / inliers, rng)
    y = add_uniform_noise(y, (n - inliers) / inliers, rng)
    return PointCloud(x.points[:n]), PointCloud(y.points[:n])


def fragment_pair(p, n=4096):
    """BASELINE configs[4] pair p: a 3DMatch-fragment-sized pair (SURVEY
    §8(d) C5) -- ``blob`` for even p, ``bumped_box`` for odd p, n points,
    misaligned by a random rigid motion of <= 60 deg / 0.1, seeded with
    100000 + p (so any shard of the batch regenerates its own pairs)."""
    rng = rng_from_seed(100000 + p)
    x = blob(n, rng) if p % 2 == 0 else bumped_box(n, rng)
    return x, misalign(x, random_rigid(rng, np.deg2rad(60), 0.1))


def configs2_pair(n=1_000_000, seed=3):
    """BASELINE configs[2]: the 1M x 1M pair --
    ``blob(n)`` and its misaligned copy (<= 60 deg / 0.1), PCG64 seed 3."""
    rng = rng_from_seed(seed)
    x = blob(n, rng)
    gt = random_rigid(rng, np.deg2rad(60), 0.1)
    return x, misalign(x, gt)


def configs1_pair(n=100_000, seed=2):
    """BASELINE configs[1]: a LiDAR-scan-shaped pair -- the
    street scan and its copy moved by <= 10 deg / 1 m, PCG64 seed 2."""
    rng = rng_from_seed(seed)
    x = lidar_scan(n, rng)
    gt = random_rigid(rng, np.deg2rad(10), 1.0)
    return x, misalign(x, gt), gt


def configs3_pair(n=200_000, seed=4):
    """BASELINE configs[3]: the 40%-overlap pair with 5% outliers and
    inhomogeneous density, template misaligned <= 60 deg."""
    rng = rng_from_seed(seed)
    x, y0 = partial_overlap(n, rng)
    gt = random_rigid(rng, np.deg2rad(60), 0.1)
    return x, misalign(y0, gt), gt
