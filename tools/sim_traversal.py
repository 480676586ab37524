"""CPU model of the warp traversal schemes (design tool, not product code).
Counts warp steps / window refills for the exact-MAC stackless traversal on
the mirrored-preorder tree, for Morton-ordered 32-query warps."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from numba import njit

from oracle import oracle as orc
from paper_2009_14005_b200 import synth


def mirror_layout(t):
    n = t.node_count
    ch = t.children
    depth = t.depth
    skip = np.empty(n, np.int64)
    for x in range(n - 1, -1, -1):
        kids = ch[x][ch[x] >= 0]
        skip[x] = x + 1 if len(kids) == 0 else skip[kids.max()]
    mir = depth + n - skip
    size = skip - np.arange(n)
    com = np.empty((n, 3))
    l2 = np.empty(n)
    sk = np.empty(n, np.int64)
    leaf = (ch < 0).all(axis=1)
    com[mir] = t.com
    l2[mir] = np.where(leaf, -np.inf, t.length ** 2)
    sk[mir] = mir + size
    return com, l2, sk


@njit(cache=True)
def sim(com, l2, sk, q, theta2, W):
    n_nodes = len(l2)
    m = len(q)
    nw = m // 32
    steps_min = 0
    refill_min = 0
    outer = 0
    inner = 0
    visits = 0
    cur = np.zeros(32, np.int64)
    for w in range(nw):
        # scheme A: warp-min with window
        for l in range(32):
            cur[l] = 0
        wbase = -10**9
        while True:
            n = cur.min()
            if n >= n_nodes:
                break
            if n - wbase >= W or n < wbase:
                wbase = n
                refill_min += 1
            steps_min += 1
            for l in range(32):
                if cur[l] == n:
                    qi = w * 32 + l
                    d2 = 0.0
                    for k in range(3):
                        dk = q[qi, k] - com[n, k]
                        d2 += dk * dk
                    visits += 1
                    if l2[n] < theta2 * d2:
                        cur[l] = sk[n]
                    else:
                        cur[l] = n + 1
        # scheme B: windowed independent lanes
        for l in range(32):
            cur[l] = 0
        while True:
            n = cur.min()
            if n >= n_nodes:
                break
            outer += 1
            wend = min(n + W, n_nodes)
            it = 0
            while True:
                moved = False
                for l in range(32):
                    c = cur[l]
                    if c < wend:
                        moved = True
                        qi = w * 32 + l
                        d2 = 0.0
                        for k in range(3):
                            dk = q[qi, k] - com[c, k]
                            d2 += dk * dk
                        if l2[c] < theta2 * d2:
                            cur[l] = sk[c]
                        else:
                            cur[l] = c + 1
                if not moved:
                    break
                it += 1
            inner += it
    return steps_min, refill_min, outer, inner, visits


@njit(cache=True)
def sim_groups(com, l2, sk, q, theta2, G):
    """warp-min traversal with the 32 lanes split into 32/G independent groups
    of G lanes (each with its own minimum cursor): warp iterations = max over
    the groups of their union steps."""
    n_nodes = len(l2)
    nw = len(q) // 32
    total = 0
    cur = np.zeros(32, np.int64)
    for w in range(nw):
        worst = 0
        for g0 in range(0, 32, G):
            for l in range(G):
                cur[l] = 0
            steps = 0
            while True:
                n = cur[:G].min()
                if n >= n_nodes:
                    break
                steps += 1
                for l in range(G):
                    if cur[l] == n:
                        qi = w * 32 + g0 + l
                        d2 = 0.0
                        for k in range(3):
                            dk = q[qi, k] - com[n, k]
                            d2 += dk * dk
                        if l2[n] < theta2 * d2:
                            cur[l] = sk[n]
                        else:
                            cur[l] = n + 1
            worst = max(worst, steps)
        total += worst
    return total


@njit(cache=True)
def sim_thread(com, l2, sk, q, theta2):
    """independent per-lane traversal: warp steps = max lane visits; also the
    number of distinct nodes (and 128-B lines of 24-B records) per step."""
    n_nodes = len(l2)
    nw = len(q) // 32
    steps = 0
    distinct = 0
    lines = 0
    cur = np.zeros(32, np.int64)
    for w in range(nw):
        for l in range(32):
            cur[l] = 0
        while True:
            alive = 0
            nodes = np.empty(32, np.int64)
            for l in range(32):
                c = cur[l]
                if c < n_nodes:
                    nodes[alive] = c
                    alive += 1
                    qi = w * 32 + l
                    d2 = 0.0
                    for k in range(3):
                        dk = q[qi, k] - com[c, k]
                        d2 += dk * dk
                    if l2[c] < theta2 * d2:
                        cur[l] = sk[c]
                    else:
                        cur[l] = c + 1
            if alive == 0:
                break
            steps += 1
            u = np.unique(nodes[:alive])
            distinct += len(u)
            lines += len(np.unique((u * 24) // 128))
    return steps, distinct, lines


def hilbert3(X, bits):
    """3-D Hilbert index of integer coordinates (Skilling's transpose)."""
    X = X.copy()
    M = 1 << (bits - 1)
    Q = M
    while Q > 1:
        P = Q - 1
        for i in range(3):
            m = (X[:, i] & Q) != 0
            X[m, 0] ^= P
            nm = ~m
            t = (X[nm, 0] ^ X[nm, i]) & P
            X[nm, 0] ^= t
            X[nm, i] ^= t
        Q >>= 1
    for i in range(1, 3):
        X[:, i] ^= X[:, i - 1]
    t = np.zeros(len(X), dtype=X.dtype)
    Q = M
    while Q > 1:
        m = (X[:, 2] & Q) != 0
        t[m] ^= Q - 1
        Q >>= 1
    for i in range(3):
        X[:, i] ^= t
    idx = np.zeros(len(X), dtype=np.int64)
    for b in range(bits - 1, -1, -1):
        for i in range(3):
            idx = (idx << 1) | ((X[:, i] >> b) & 1)
    return idx


def main(n=1_000_000, nq=16384, theta=0.5):
    rng = synth.rng_from_seed(3)
    x = synth.blob(n, rng)
    y = synth.misalign(x, synth.random_rigid(rng, np.deg2rad(60), 0.1))
    xn, yn, _ = orc.normalize_pair(x.points, y.points, -5.0, 5.0)
    sx = orc.niv_masses(xn, 16, -5.0, 5.0, 20)
    sy = orc.niv_masses(yn, 16, -5.0, 5.0, 20)
    mx, _ = orc.rescale(sx, sy, 0.1, 0.2)
    t = orc.tree_build(xn, mx, 20)
    com, l2, sk = mirror_layout(t)
    # Morton order of the template (same keys as the device: 21 bits/axis)
    lo, hi = yn.min(0), yn.max(0)
    qq = np.clip((yn - lo) / (hi - lo), 0, 1)
    qi = (qq * 2097151).astype(np.uint64)

    def spread(v):
        v = v & np.uint64(0x1fffff)
        v = (v | (v << np.uint64(32))) & np.uint64(0x1f00000000ffff)
        v = (v | (v << np.uint64(16))) & np.uint64(0x1f0000ff0000ff)
        v = (v | (v << np.uint64(8))) & np.uint64(0x100f00f00f00f00f)
        v = (v | (v << np.uint64(4))) & np.uint64(0x10c30c30c30c30c3)
        v = (v | (v << np.uint64(2))) & np.uint64(0x1249249249249249)
        return v
    key = (spread(qi[:, 0]) << np.uint64(2)) | (spread(qi[:, 1]) << np.uint64(1)) | spread(qi[:, 2])
    order = np.argsort(key, kind="stable")
    if os.environ.get("SIM_ORDER"):  # Morton vs Hilbert 32-query warps, union overhead
        hord = np.argsort(hilbert3(np.clip((qq * 1023).astype(np.int64), 0, 1023), 10),
                          kind="stable")
        h16 = np.argsort(hilbert3(np.clip((qq * 65535).astype(np.int64), 0, 65535), 16),
                         kind="stable")
        xl, xh = xn.min(0), xn.max(0)  # the reference cloud's box (the tree's cells)
        qr = np.clip((yn - xl) / (xh - xl), 0, 1)
        hx = np.argsort(hilbert3(np.clip((qr * 1023).astype(np.int64), 0, 1023), 10),
                        kind="stable")
        orders = (("morton", order), ("hilbert", hord), ("hilbert16", h16), ("hilbert_refbox", hx))
        if os.environ.get("SIM_ORDER") == "groups":
            for frac in (0.25, 0.5, 0.75):
                st0 = int(len(hord) * frac)
                qs = np.ascontiguousarray(yn[hord[st0:st0 + nq]])
                r = [sim_groups(com, l2, sk, qs, theta * theta, G) / (nq / 32) for G in (32, 16, 8)]
                print(f"hilbert @{frac}: warp iterations per warp  G=32 {r[0]:.0f}  G=16 {r[1]:.0f}  G=8 {r[2]:.0f}")
            return
        if os.environ.get("SIM_ORDER") == "2":
            orders = orders[1:]
        for name, o in orders:
            for frac in (0.25, 0.5, 0.75):
                st0 = int(len(o) * frac)
                qs = np.ascontiguousarray(yn[o[st0:st0 + nq]])
                a = sim(com, l2, sk, qs, theta * theta, 32)
                print(f"{name} @{frac}: steps/warp {a[0]/(nq/32):.0f} visits/q {a[4]/nq:.0f} "
                      f"union {a[0]/(nq/32)/(a[4]/nq):.3f}")
        return
    start = len(order) // 2
    sel = order[start:start + nq]
    q = np.ascontiguousarray(yn[sel])
    for W in (32, 64, 128, 256):
        t0 = time.time()
        a = sim(com, l2, sk, q, theta * theta, W)
        print(f"W={W}: warp-min steps/warp {a[0]/(nq/32):.0f} refills/warp {a[1]/(nq/32):.0f} | "
              f"windowed outer/warp {a[2]/(nq/32):.0f} inner/warp {a[3]/(nq/32):.0f} | "
              f"visits/q {a[4]/nq:.0f}  ({time.time()-t0:.1f}s)")
    if os.environ.get("SIM_THREAD"):
        b = sim_thread(com, l2, sk, q, theta * theta)
    else:
        return
    print(f"per-thread: steps/warp {b[0]/(nq/32):.0f}  distinct nodes/step {b[1]/b[0]:.2f} "
          f"128B lines/step {b[2]/b[0]:.2f}")


if __name__ == "__main__":
    main(*(int(v) for v in sys.argv[1:3]))
