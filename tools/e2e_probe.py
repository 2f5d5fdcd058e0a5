"""Profiling driver (not part of the product): per-call wall time of the host-pointer
matvec (the e2e path) and of its pieces, for the cached config-3 matrix."""
import os, pickle, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2308_10960_b200.hmatrix import HMatrix  # noqa: E402
from paper_2308_10960_b200._lib import check, lib  # noqa: E402

flat = pickle.load(open(sys.argv[1], "rb"))
flat.blob = torch.as_tensor(flat.blob).cuda()
H = HMatrix(flat)
n = flat.n_rows
xh = torch.randn(n, dtype=torch.float64).pin_memory()
yh = torch.zeros(n, dtype=torch.float64).pin_memory()
x = xh.cuda(); y = torch.zeros_like(x)
for _ in range(5):
    check(lib().hcmx_gpu_hmat_matvec(H._h, 1.0, xh.data_ptr(), 0.0, yh.data_ptr(), 0))
N = 100
t = time.perf_counter()
for _ in range(N):
    check(lib().hcmx_gpu_hmat_matvec(H._h, 1.0, xh.data_ptr(), 0.0, yh.data_ptr(), 0))
e2e = (time.perf_counter() - t) / N
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(N):
    H.matvec_device(1.0, x, 0.0, y)
    torch.cuda.synchronize()
dev_sync = (time.perf_counter() - t) / N
t = time.perf_counter()
for _ in range(N):
    x.copy_(xh, non_blocking=True); yh.copy_(y, non_blocking=True); torch.cuda.synchronize()
copies = (time.perf_counter() - t) / N
print(f"e2e {e2e*1e6:.1f} us  device+sync {dev_sync*1e6:.1f} us  copies+sync {copies*1e6:.1f} us")
