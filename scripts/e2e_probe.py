"""Host-pointer sigma (pinned buffers) vs device sigma at a config; with
DETCI_PIPE_DEBUG=1 the pipelined path prints its phase split."""
import sys
import time
import ctypes as C
import numpy as np
import torch
sys.path.insert(0, '/root/repo')
from paper_2601_16169_b200 import _lib, detci, synth
cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
ints, a, b = synth.synthetic_system(cfg)
basis = detci.GpuBasis(ints.norbs, a, b, ints.core, ints.h1, ints.eri)
lib = _lib.load()
x = torch.from_numpy(synth.random_vector(basis.dimension(), 11)).pin_memory()
y = torch.empty_like(x).pin_memory()
dx, dy = x.cuda(), torch.empty_like(x).cuda()
for rep in range(4):
    torch.cuda.synchronize()
    t0 = time.time()
    code = lib.detci_gpu_sigma(basis.handle, x.data_ptr(), y.data_ptr(), None)
    assert code == 0, (code, lib.detci_gpu_last_error(basis.handle))
    t1 = time.time()
    tm = _lib.Timings()
    assert lib.detci_gpu_sigma_device(basis.handle, dx.data_ptr(), dy.data_ptr(), None) == 0
    torch.cuda.synchronize()
    t2 = time.time()
    print(f"{cfg} host sigma {1e3*(t1-t0):.2f} ms, device sigma {1e3*(t2-t1):.2f} ms", flush=True)
