"""CPU stand-in for the libfga session, used only by the multi-process tests.

It restates, in numpy on top of the oracle, exactly what the device session
computes per shard: the pending-transform prologue, forces + Euler-Cromer
step, the shifted Kabsch moments written into the 18-double sums buffer, and
the fp64 update (rigid.cu k_update).  With it, paper_2009_14005_b200.distributed
.run_sharded -- the real collective schedule -- runs over gloo on CPU.
"""

import numpy as np
import torch

from oracle import oracle as orc

SUMS = 18


class NumpyShardBackend:
    def __init__(self, x, y, params, rank, world, theta=None):
        p = params
        self.p = p
        a, b = p.norm_range
        xn, yn, self.ctx = orc.normalize_pair(x, y, a, b)
        sx = orc.niv_masses(xn, p.rho, a, b, p.max_depth)
        sy = orc.niv_masses(yn, p.rho, a, b, p.max_depth)
        mx, my = orc.rescale(sx, sy, p.dt, p.eta)
        self.xn, self.mx = xn, mx
        self.tree = orc.tree_build(xn, mx, p.max_depth)
        m = len(yn)
        lo, hi = m * rank // world, m * (rank + 1) // world
        self.pos = yn[lo:hi].copy()
        self.vel = np.zeros_like(self.pos)
        self.mq = my[lo:hi].copy()
        self.m_total = m
        self.Rp, self.tp = np.eye(3), np.zeros(3)
        self.Racc, self.tacc = np.eye(3), np.zeros(3)
        self.shift = yn.mean(axis=0)
        self.iter = 0
        self.done = False
        self.converged = False
        self.deltas, self.traj = [], []
        self.gpe_vals = {}
        self.applied = False
        self.sums = torch.zeros(SUMS, dtype=torch.float64)

    # --- pieces of the device session
    def forces(self):
        self.sums.zero_()
        if self.done:
            return
        self.pos = self.pos @ self.Rp.T + self.tp
        self.vel = self.vel @ self.Rp.T
        p = self.p
        grav, visits, acc = orc.bh_forces(self.tree, self.pos, self.mq, p.theta, p.G, p.epsilon)
        vp, d = orc.step(self.pos, self.vel, self.mq, grav, p.dt, p.eta)
        self.vel = vp
        u = self.pos - self.shift
        w = self.pos + d - self.shift
        s = np.zeros(SUMS)
        s[0:3] = u.sum(0)
        s[3:6] = w.sum(0)
        s[6:15] = (w.T @ u).ravel()
        s[15] = acc.sum()
        s[16] = visits.sum()
        self.sums.copy_(torch.from_numpy(s))

    def update(self):
        if self.done:
            return
        s = self.sums.numpy()
        M = float(self.m_total)
        mu_u, mu_w = s[0:3] / M, s[3:6] / M
        C = s[6:15].reshape(3, 3) - M * np.outer(mu_w, mu_u)
        U, S, Vt = np.linalg.svd(C)
        sgn = np.sign(np.linalg.det(U @ Vt)) or 1.0
        R = U @ np.diag([1.0, 1.0, sgn]) @ Vt
        mu_y, mu_d = mu_u + self.shift, mu_w + self.shift
        t = mu_d - R @ mu_y
        Ra, ta = R @ self.Racc, t + R @ self.tacc
        delta = float(((Ra - self.Racc) ** 2).sum() + ((ta - self.tacc) ** 2).sum())
        self.Rp, self.tp, self.Racc, self.tacc, self.shift = R, t, Ra, ta, mu_d
        self.deltas.append(delta)
        self.traj.append(np.hstack([Ra, ta[:, None]]))
        self.iter += 1
        if delta < self.p.conv_tol:
            self.converged = self.done = True
        elif self.iter >= self.p.max_iters:
            self.done = True

    def gpe(self):
        self.sums.zero_()
        p = self.p
        part = orc.gpe(self.pos, self.mq, self.xn, self.mx, 1.0, p.epsilon) * -1.0
        self.sums[17] = part

    def take_gpe(self):
        return -self.p.G * float(self.sums[17])

    def set_gpe(self, which, v):
        self.gpe_vals[which] = v

    def apply_pending(self):
        if not self.applied:
            self.pos = self.pos @ self.Rp.T + self.tp
            self.applied = True

    def poll(self):
        return self.done, self.iter

    def finish(self):
        return dict(R=self.Racc, t=self.tacc, iterations=self.iter, converged=self.converged,
                    deltas=np.array(self.deltas), traj=np.array(self.traj),
                    gpe_initial=self.gpe_vals.get(0), gpe_final=self.gpe_vals.get(1))
