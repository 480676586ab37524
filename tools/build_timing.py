"""Tree build wall time (CUDA events, L2 flushed) for a blob of n points:
    python tools/build_timing.py [n ...]   (FGA_LIB_PATH selects the library)"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2009_14005_b200 import _native as N
from paper_2009_14005_b200 import synth

dev = torch.device("cuda", 0)
c = N.Context(0)
st = torch.cuda.current_stream()
c.set_stream(st.cuda_stream)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for n in [int(a) for a in sys.argv[1:]] or [1_000_000, 16_000_000]:
    pts = torch.from_numpy(np.ascontiguousarray(synth.blob(n, synth.rng_from_seed(3)).points)).to(dev)
    ms = torch.ones(n, dtype=torch.float64, device=dev)
    nn = N._i64(0)
    ts = []
    for r in range(13):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        N.check(N.lib().fga_tree_build_dev(c.handle, pts.data_ptr(), ms.data_ptr(), n, 20,
                                           ctypes.byref(nn)))
        b.record(st)
        torch.cuda.synchronize()
        if r >= 3:
            ts.append(a.elapsed_time(b))
    print(f"n={n} nodes={nn.value} build median {np.median(ts):.3f} ms (min {min(ts):.3f})")
