"""RLS stream latency probe: one / many prequential streams of L samples
through intf_rls_streams (k_rls_g8), CUDA-event timed."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2512_18725_b200 import _abi  # noqa: E402

L = _abi.load()
for n_streams, ln in [(1, 720), (4, 720), (64, 720), (10000, 73), (10000, 300)]:
    rng = np.random.default_rng(0)
    n = n_streams * ln
    X = torch.tensor(rng.uniform(0, 1, size=(n, 6)), device="cuda")
    y = torch.tensor(rng.uniform(1, 2, size=n), device="cuda")
    off = torch.arange(0, n + 1, ln, dtype=torch.int64, device="cuda")
    p0 = torch.zeros(n_streams, 7, dtype=torch.float64, device="cuda")
    P0 = (100.0 * torch.eye(7, dtype=torch.float64, device="cuda")).repeat(n_streams, 1, 1).contiguous()
    lam = torch.full((n_streams,), 0.99, dtype=torch.float64, device="cuda")
    pred = torch.empty(n, dtype=torch.float64, device="cuda")
    st = torch.zeros(n_streams, dtype=torch.int32, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    ts = []
    for rep in range(4):
        p, P = p0.clone(), P0.clone()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _abi.check(L.intf_rls_streams(X.data_ptr(), y.data_ptr(), off.data_ptr(), n_streams, lam.data_ptr(),
                                      p.data_ptr(), P.data_ptr(), pred.data_ptr(), st.data_ptr(), s), "rls")
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = min(ts[1:])
    print(f"streams {n_streams:6d} x {ln:4d}: {ms:.3f} ms  {1e3 * ms / ln:.3f} us/update on the chain")
