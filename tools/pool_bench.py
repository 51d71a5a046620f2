"""Pooled forward (k_pool / k_pool1 via fc_pool_rows) on synthetic multi-hot bags:
HBM GB/s against algorithmic bytes for bag sizes 1..32 (rows resident in HBM)."""
import ctypes, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2208_05321_b200 import _lib
lib = _lib.load()
dev = torch.device("cuda", 0)
U, D, N = 500_000, 128, 425_984
rows = torch.randn(U, D, device=dev)
g = torch.Generator(device=dev); g.manual_seed(0)
inv = torch.randint(0, U, (N,), device=dev, generator=g, dtype=torch.int32)
psw = torch.rand(N, device=dev)
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
for L in (1, 2, 4, 8, 16, 32):
    for mode, w in (("sum", None), ("mean", psw)):
        nb = N // L
        off = None if L == 1 else torch.arange(0, N, L, device=dev, dtype=torch.int64)
        out = torch.empty(nb, D, device=dev)
        def run():
            rc = lib.fc_pool_rows(ctypes.c_void_p(rows.data_ptr()), D, ctypes.c_void_p(inv.data_ptr()), N,
                                  ctypes.c_void_p(0 if off is None else off.data_ptr()), 0 if off is None else 8, nb, 0,
                                  ctypes.c_void_p(0 if w is None else w.data_ptr()), 0 if mode == "sum" else 1,
                                  ctypes.c_void_p(out.data_ptr()), st)
            assert rc == 0
        for _ in range(3): run()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); e0.record()
        for _ in range(20): run()
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 20
        by = N * (4 * D + 4 + (4 if w is not None else 0)) + nb * (4 * D + (8 if off is not None else 0))
        print(f"L={L:2d} {mode:4s} psw={w is not None}: {ms*1e3:7.1f} us  {by / ms / 1e6:7.0f} GB/s")
