"""Experiment (tools/): windowed refit timing (intf_ols_windows) at several
window sizes; run under ncu for the per-kernel split."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2512_18725_b200 import _abi

L = _abi.load()
n = 1 << 24
X = torch.rand(n, 6, dtype=torch.float64, device="cuda")
y = torch.rand(n, dtype=torch.float64, device="cuda")
for W in (8, 32, 64, 100, 256, 1024):
    nw = (n + W - 1) // W
    st = torch.empty(nw * 56, dtype=torch.float64, device="cuda")
    pr = torch.empty(nw * 7, dtype=torch.float64, device="cuda")
    inf = torch.empty(nw * 3, dtype=torch.int32, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    f = lambda: _abi.check(L.intf_ols_windows(X.data_ptr(), y.data_ptr(), n, W, None if W % 8 == 0 else st.data_ptr(),
                                              pr.data_ptr(), inf.data_ptr(), s), "w")
    for _ in range(3):
        f()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        f()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"W={W}: {ms:.3f} ms, {nw / ms * 1e3:.3e} fits/s, {56 * n / ms / 1e6:.0f} GB/s")
