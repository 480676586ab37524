"""1M configs[2] BH iteration time (the bench's main leg, CUDA events, L2
flushed) + FP32 force accuracy on 16,384 sampled queries vs the oracle, for
the library FGA_LIB_PATH points at (A/B tool).  usage: python tools/iter_timing.py [steps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2009_14005_b200 as fga
from paper_2009_14005_b200 import bhtree, synth
from paper_2009_14005_b200.engine import Session

K = int(sys.argv[1]) if len(sys.argv) > 1 else 20
n = int(os.environ.get("FGA_N", "1000000"))
x, y = synth.configs2_pair(n)
p = fga.default_params().replace(theta=0.5, G=66.7 * (2000.0 / n) ** 0.5, conv_tol=1e-300,
                                 max_iters=K + 5)
dev = torch.device("cuda", 0)
xt = torch.from_numpy(np.array(x.points)).to(dev)
yt = torch.from_numpy(np.array(y.points)).to(dev)
st = torch.cuda.current_stream()
prec = os.environ.get("FGA_PREC", "fp32")
s = Session(None, None, p, fga.RegisterOptions(compute_gpe=False, precision=prec), stream=st.cuda_stream,
            device_inputs=(xt.data_ptr(), n, yt.data_ptr(), n))
for _ in range(3):
    s.forces()
    s.update()
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
torch.cuda.synchronize()
for k in range(K):
    flush.zero_()
    ev[k][0].record(st)
    s.forces()
    ev[k][1].record(st)
    s.update()
torch.cuda.synchronize()
ms = np.array([a.elapsed_time(b) for a, b in ev])
res = s.finish()
inter = res.interactions[3:3 + K].mean()
line = f"force pass {ms.mean():.3f} ms (min {ms.min():.3f})  {inter / ms.mean() * 1e3:.4g} inter/s"
if os.environ.get("FGA_ACC", "1") == "1" and prec == "fp32":
    from oracle import oracle as orc
    xn, yn, mx, my, _ = orc.setup(x.points, y.points)
    ot = orc.tree_build(xn, mx, 20)
    idx = np.sort(np.random.default_rng(0).choice(n, 16384, replace=False))
    of, ov, oa = orc.bh_forces(ot, yn[idx], my[idx], 0.5, p.G, p.epsilon)
    t = bhtree.build(fga.PointCloud(xn), mx, 20)
    f, v, a = bhtree.bh_forces(t, yn[idx], my[idx], p, precision="fp32", return_accepted=True)
    rel = np.linalg.norm(f - of, axis=1) / np.linalg.norm(of, axis=1)
    line += (f"  | visits equal {np.array_equal(v, ov) and np.array_equal(a, oa)}  rel max "
             f"{rel.max():.2e} p99 {np.quantile(rel, 0.99):.2e}")
print(os.path.basename(os.environ.get("FGA_LIB_PATH", "libfga.so")), prec, line, flush=True)
