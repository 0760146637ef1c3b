"""Per-vector sigma time for blocks of M = 1, 2, 4 vectors (device buffers)."""
import ctypes as C
import sys
import time
import numpy as np
import torch
sys.path.insert(0, '/root/repo')
from paper_2601_16169_b200 import _lib, detci, synth
cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
ints, a, b = synth.synthetic_system(cfg)
basis = detci.GpuBasis(ints.norbs, a, b, ints.core, ints.h1, ints.eri)
lib = _lib.load()
n = basis.local_dim
xs = [torch.from_numpy(synth.random_vector(n, 11 + i)).cuda() for i in range(4)]
ys = [torch.empty_like(xs[0]) for _ in range(4)]
ref = []
for m in (1, 2, 4):
    px = (C.c_void_p * m)(*[t.data_ptr() for t in xs[:m]])
    py = (C.c_void_p * m)(*[t.data_ptr() for t in ys[:m]])
    args = (basis.handle, C.cast(px, C.POINTER(C.c_void_p)), C.cast(py, C.POINTER(C.c_void_p)), m)
    assert lib.detci_gpu_sigma_block(*args) == 0
    torch.cuda.synchronize()
    t0 = time.time()
    for _ in range(3):
        assert lib.detci_gpu_sigma_block(*args) == 0
    torch.cuda.synchronize()
    dt = (time.time() - t0) / 3
    if m == 1:
        ref = ys[0].cpu().numpy()
    err = float(np.max(np.abs(ys[0].cpu().numpy() - ref) / np.maximum(1, np.abs(ref))))
    print(f"{cfg} M={m}: {dt*1e3:.1f} ms per block, {dt/m*1e3:.1f} ms per vector, rel err vs M=1 {err:.2e}", flush=True)
