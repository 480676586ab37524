"""configs[4] batch on device-resident clouds (fga_register_batch_dev, CUDA
events): pairs/s of the kernel path alone.  usage: python tools/batch_kernel_timing.py [P]"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2009_14005_b200 as fga
from paper_2009_14005_b200 import _native as N
from paper_2009_14005_b200 import synth

P = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
pairs = [synth.fragment_pair(p) for p in range(P)]
xoff = np.zeros(P + 1, np.int64)
yoff = np.zeros(P + 1, np.int64)
xoff[1:] = np.cumsum([len(x) for x, _ in pairs])
yoff[1:] = np.cumsum([len(y) for _, y in pairs])
dev = torch.device("cuda", 0)
Xd = torch.from_numpy(np.concatenate([x.points for x, _ in pairs])).to(dev)
Yd = torch.from_numpy(np.concatenate([y.points for _, y in pairs])).to(dev)
xo = torch.from_numpy(xoff).to(dev)
yo = torch.from_numpy(yoff).to(dev)
res = torch.empty(P * ctypes.sizeof(N.CPairResult), dtype=torch.uint8, device=dev)
cp = N.make_params(fga.default_params())
co = fga.registration._c_options(fga.RegisterOptions(), None, None)
c = N.context(0)
c.set_stream(torch.cuda.current_stream().cuda_stream)
L = N.lib()


def run():
    N.check(L.fga_register_batch_dev(c.handle, Xd.data_ptr(), xo.data_ptr(), Yd.data_ptr(),
                                     yo.data_ptr(), P, 4096, 4096, 3, ctypes.byref(cp),
                                     ctypes.byref(co), res.data_ptr(), None))


run()
ts = []
for _ in range(3):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    run()
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b) / 1e3)
out = (N.CPairResult * P).from_buffer_copy(res.cpu().numpy().tobytes())
its = np.array([r.iterations for r in out])
st = np.array([r.status for r in out])
R = np.array([r.R for r in out])
print(f"mode={os.environ.get('FGA_BATCH_WIDE', 'auto')} {P} pairs kernel {min(ts):.4f} s -> "
      f"{P / min(ts):.0f} pairs/s; iterations median {np.median(its)} max {its.max()}; "
      f"failed {int((st != 0).sum())}; R checksum {np.abs(R).sum():.10f}")
