"""ncu driver for the tree build (fga_tree_build_dev): one warm-up build and
one profiled build of an N-point blob.  Not a benchmark."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2009_14005_b200 import _native as N
from paper_2009_14005_b200 import synth

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16_000_000
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
dev = torch.device("cuda", 0)
pts = torch.from_numpy(synth.blob(n, synth.rng_from_seed(3)).points).to(dev)
ms = torch.ones(n, dtype=torch.float64, device=dev)
c = N.Context(0)
c.set_stream(torch.cuda.current_stream().cuda_stream)
nn = N._i64(0)
for _ in range(reps):
    N.check(N.lib().fga_tree_build_dev(c.handle, pts.data_ptr(), ms.data_ptr(), n, 20,
                                       ctypes.byref(nn)))
torch.cuda.synchronize()
print("nodes", nn.value)
