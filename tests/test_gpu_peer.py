"""The owner-side fused return exchange (fc_pool_to_peers): rows written straight into
requesters' buffers through peer pointers. One GPU here, so (1) several local buffers
stand in for W peers to check the segment -> buffer/offset addressing, (2) two
processes on the same GPU exercise the CUDA-IPC path (fc_ipc_handle / fc_ipc_open),
(3) RowShardedEmbedding(peer_rows=...) trains through NCCL at world 1 like the dense
reference."""

import ctypes

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

import paper_2208_05321_b200 as fc  # noqa: E402
from paper_2208_05321_b200 import _lib  # noqa: E402

lib = _lib.load()


def _stack(num_ids=5000, dim=16, cap=1000):
    idx = fc.IdxMap(np.arange(num_ids), np.arange(num_ids))
    rows = np.random.default_rng(1).standard_normal((num_ids, dim)).astype(np.float32)
    st = fc.CacheStack(idx, fc.SlowTierStore(rows.copy()), fc.FastTierStore(np.zeros((cap, dim), np.float32)),
                       fc.Transmitter())
    return st, rows


def test_pool_to_peers_addressing():
    st, rows = _stack()
    ids = np.random.default_rng(2).integers(0, 5000, 900)
    p = st.prepare(ids, 0)
    n, W = ids.size, 3
    seg = np.array([0, 250, 600, n], dtype=np.int64)          # received ids of requesters 0, 1, 2
    off = np.array([7, 0, 31], dtype=np.int64)               # where this owner's rows start in each
    bufs = [torch.zeros((off[r] + seg[r + 1] - seg[r] + 5, 16), device="cuda") for r in range(W)]
    dst = torch.tensor([b.data_ptr() for b in bufs], dtype=torch.int64, device="cuda")
    seg_d = torch.from_numpy(seg).cuda()
    off_d = torch.from_numpy(off).cuda()
    dc = st.device
    rc = lib.fc_pool_to_peers(dc.h, ctypes.c_void_p(p.d_unique_slots.data_ptr()),
                              ctypes.c_void_p(p.d_inverse.data_ptr()),
                              n, ctypes.c_void_p(seg_d.data_ptr()), W, ctypes.c_void_p(dst.data_ptr()),
                              ctypes.c_void_p(off_d.data_ptr()), dc.stream())
    assert rc == _lib.OK
    torch.cuda.synchronize()
    for r in range(W):
        got = bufs[r].cpu().numpy()
        want = rows[ids[seg[r]:seg[r + 1]]]
        assert np.array_equal(got[off[r]:off[r] + want.shape[0]], want), r
        assert not got[:off[r]].any() and not got[off[r] + want.shape[0]:].any(), r


def _peer_child(conn):
    import torch as t

    from paper_2208_05321_b200 import _lib as L

    lb = L.load()
    st, rows = _stack()
    ids = np.arange(100, 400)
    p = st.prepare(ids, 0)
    handle = conn.recv()
    ptr = ctypes.c_void_p()
    buf = (ctypes.c_ubyte * 128).from_buffer_copy(handle)
    assert lb.fc_ipc_open(buf, 0, ctypes.byref(ptr)) == L.OK
    dst = t.tensor([ptr.value], dtype=t.int64, device="cuda")
    seg = t.tensor([0, ids.size], dtype=t.int64, device="cuda")
    off = t.tensor([10], dtype=t.int64, device="cuda")
    rc = lb.fc_pool_to_peers(st.device.h, ctypes.c_void_p(p.d_unique_slots.data_ptr()),
                             ctypes.c_void_p(p.d_inverse.data_ptr()), ids.size, ctypes.c_void_p(seg.data_ptr()), 1,
                             ctypes.c_void_p(dst.data_ptr()), ctypes.c_void_p(off.data_ptr()), st.device.stream())
    t.cuda.synchronize()
    lb.fc_ipc_close(ptr)
    conn.send(rc)


def test_pool_to_peers_over_cuda_ipc():
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    a, b = ctx.Pipe()
    proc = ctx.Process(target=_peer_child, args=(b,))
    proc.start()
    # buf sits at an offset inside its allocation (the caching allocator's case): the
    # exported handle must carry the offset for the peer to write at buf, not at the base
    big = torch.zeros((1000, 16), device="cuda")
    buf = big[300:700]
    torch.cuda.synchronize()  # the zero fill lands before the peer process writes into buf
    hd = (ctypes.c_ubyte * 128)()
    assert lib.fc_ipc_handle(ctypes.c_void_p(buf.data_ptr()), hd) == _lib.OK
    a.send(bytes(hd))
    assert a.recv() == _lib.OK
    proc.join(timeout=120)
    rows = np.random.default_rng(1).standard_normal((5000, 16)).astype(np.float32)
    got = buf.cpu().numpy()
    assert np.array_equal(got[10:310], rows[100:400]) and not got[:10].any()
    assert not big[:300].cpu().numpy().any()  # nothing written at the allocation's base


def test_row_sharded_peer_rows_nccl_world1_matches_dense():
    import torch.distributed as dist

    from paper_2208_05321_b200.distributed import CudaShard, RowShardedEmbedding, shard_rows_for_rank
    from paper_2208_05321_b200.store import fast_capacity, pinned_empty

    if not dist.is_initialized():
        dist.init_process_group("nccl", store=dist.HashStore(), rank=0, world_size=1)
    num_ids, dim, steps, B = 30_000, 16, 5, 4_000
    rng = np.random.default_rng(4)
    p = 1.0 / np.arange(1, num_ids + 1) ** 1.1
    trace = rng.permutation(num_ids)[rng.choice(num_ids, size=(steps, B), p=p / p.sum())]
    table = rng.uniform(-0.1, 0.1, (num_ids, dim)).astype(np.float32)
    idx = shard_rows_for_rank(np.bincount(trace.reshape(-1), minlength=num_ids), 0, 1)
    rows = pinned_empty((num_ids, dim))
    rows[...] = table[idx.id_of]
    shard = CudaShard(num_ids, dim, fast_capacity(num_ids, 0.05), rows, idx, lr=0.1, device="cuda",
                      global_num_ids=num_ids)
    mod = RowShardedEmbedding(shard, 1, 0, mode="sum", device=torch.device("cuda"), peer_rows=B)
    assert mod.peer is not None
    grads = [rng.standard_normal((B, dim)).astype(np.float32) for _ in range(steps)]
    dense = torch.nn.EmbeddingBag(num_ids, dim, mode="sum", sparse=True)
    dense.weight.data = torch.from_numpy(table.copy())
    opt = torch.optim.SGD(dense.parameters(), lr=0.1)
    ids = [torch.from_numpy(trace[s]).cuda() for s in range(steps)]
    for s in range(steps):
        out = mod(ids[s])
        want = dense(torch.from_numpy(trace[s]), torch.arange(B))
        np.testing.assert_allclose(out.detach().cpu().numpy(), want.detach().numpy(), rtol=1e-5, atol=5e-6)
        if s + 1 < steps:
            mod.prefetch(ids[s + 1])
        out.backward(torch.from_numpy(grads[s]).cuda())
        opt.zero_grad()
        want.backward(torch.from_numpy(grads[s]))
        opt.step()
    mod.flush()
    torch.cuda.synchronize()
    got = np.empty_like(table)
    got[idx.id_of] = rows
    np.testing.assert_allclose(got, dense.weight.detach().numpy(), rtol=1e-5, atol=5e-6)
    dist.destroy_process_group()


def test_gather_from_peers_addressing():
    D, W = 16, 3
    seg = np.array([0, 40, 40, 100], dtype=np.int64)   # requester 1 sends nothing
    off = np.array([5, 0, 12], dtype=np.int64)
    srcs = [torch.randn((off[r] + seg[r + 1] - seg[r] + 3, D), device="cuda") for r in range(W)]
    ptrs = torch.tensor([t.data_ptr() for t in srcs], dtype=torch.int64, device="cuda")
    out = torch.empty((100, D), device="cuda")
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    off_d, seg_d = torch.from_numpy(off).cuda(), torch.from_numpy(seg).cuda()  # kept alive across the launch
    rc = lib.fc_gather_from_peers(ctypes.c_void_p(ptrs.data_ptr()), ctypes.c_void_p(off_d.data_ptr()),
                                  ctypes.c_void_p(seg_d.data_ptr()), W, 100, D, ctypes.c_void_p(out.data_ptr()), st)
    assert rc == _lib.OK
    torch.cuda.synchronize()
    want = torch.cat([srcs[r][off[r]:off[r] + seg[r + 1] - seg[r]] for r in range(W)])
    assert torch.equal(out, want)
