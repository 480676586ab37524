"""Force-pass time of template shards of the configs[2] pair on one GPU
(shard r of N via fga_session shard_rank/shard_count) at the initial state:
the per-GPU work of an N-GPU strong-scaling run.  usage: python tools/smallm_timing.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2009_14005_b200 as fga
from paper_2009_14005_b200 import _native as N
from paper_2009_14005_b200 import synth
from paper_2009_14005_b200.engine import SUM_ACCEPTED, SUMS_LEN, Session

x, y = synth.configs2_pair()
p = fga.default_params().replace(theta=0.5, G=66.7 * (2000 / 1e6) ** 0.5, conv_tol=1e-300,
                                 max_iters=4)
dev = torch.device("cuda", 0)
xt = torch.from_numpy(np.array(x.points)).to(dev)
yt = torch.from_numpy(np.array(y.points)).to(dev)
st = torch.cuda.current_stream()
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
ALL = os.environ.get("SMALLM_ALL")  # e.g. "2,4,8": every shard of those counts
shards = ([(r, n) for n in map(int, ALL.split(",")) for r in range(n)] if ALL else
          ((0, 1), (0, 2), (0, 4), (0, 8), (3, 8), (7, 8)))
for shard in shards:
    s = Session(None, None, p, fga.RegisterOptions(compute_gpe=False), shard_rank=shard[0],
                shard_count=shard[1], stream=st.cuda_stream,
                device_inputs=(xt.data_ptr(), len(x), yt.data_ptr(), len(y)), ctx=N.Context(0))
    sums = torch.zeros(SUMS_LEN, dtype=torch.float64, device=dev)
    s.bind_sums(sums.data_ptr())
    s.checkpoint()
    ts = []
    for k in range(6):
        s.restore()
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        s.forces()
        b.record(st)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
        s.update()
    t = np.mean(ts[2:])
    inter = sums[SUM_ACCEPTED].item()
    print(os.environ.get("FGA_BH_BLOCK", "128"), shard, s.m_local, "ms %.3f" % t,
          "inter/s %.4g" % (inter / t * 1e3), flush=True)
    s.finish()
