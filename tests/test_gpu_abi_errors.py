"""The C ABI's error contract (include/freqcache_b200.h), called directly through
ctypes the way a reference-side binding would: status codes for
bad arguments, validation errors before any mutation, and the prefetch pipeline's
sequencing rules."""

import ctypes

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from paper_2208_05321_b200 import _lib  # noqa: E402
from paper_2208_05321_b200.store import pinned_empty  # noqa: E402

lib = _lib.load()


def make(num_ids=1000, cap=100, dim=8):
    h = ctypes.c_void_p()
    assert lib.fc_create(num_ids, cap, dim, 0, 0, 0, 1 << 20, 0, ctypes.byref(h)) == _lib.OK
    rows = pinned_empty((num_ids, dim))
    rows[...] = np.arange(num_ids * dim, dtype=np.float32).reshape(num_ids, dim)
    rank_of = np.arange(num_ids, dtype=np.int64)
    assert lib.fc_set_idx_map(h, rank_of.ctypes.data_as(ctypes.c_void_p), None) == _lib.OK
    assert lib.fc_attach_slow_tier(h, rows.ctypes.data_as(ctypes.c_void_p), dim, None, 0) == _lib.OK
    return h, rows


def test_create_rejects_bad_geometry():
    h = ctypes.c_void_p()
    assert lib.fc_create(10, 0, 8, 0, 0, 0, 1 << 20, 0, ctypes.byref(h)) == _lib.ERR_BAD_ARG       # capacity 0
    assert lib.fc_create(10, 20, 8, 0, 0, 0, 1 << 20, 0, ctypes.byref(h)) == _lib.ERR_BAD_ARG      # capacity > ids
    assert b"capacity" in lib.fc_last_error()
    assert lib.fc_create(10, 5, 8, 0, 7, 0, 1 << 20, 0, ctypes.byref(h)) == _lib.ERR_BAD_ARG       # write_back
    assert lib.fc_create(10, 5, 8, 0, 0, 3, 1 << 20, 0, ctypes.byref(h)) == _lib.ERR_BAD_ARG       # evict_mode


def test_prepare_status_codes_and_no_mutation():
    h, _ = make()
    n = 3
    out = torch.empty(4 * n + n, dtype=torch.int32, device="cuda")
    p = [ctypes.c_void_p(out[i * n:(i + 1) * n].data_ptr()) for i in range(5)]
    info = _lib.PrepareInfo()
    bad = torch.tensor([1, 2000, 3], dtype=torch.int64, device="cuda")
    rc = lib.fc_prepare(h, ctypes.c_void_p(bad.data_ptr()), 8, n, 0, *p, None, ctypes.byref(info))
    assert rc == _lib.ERR_ID_OUT_OF_RANGE and info.bad_id == 2000 and b"2000" in lib.fc_last_error()
    assert lib.fc_free_count(h) == 100  # nothing admitted
    big = torch.arange(200, dtype=torch.int64, device="cuda")
    o2 = torch.empty(5 * 200, dtype=torch.int32, device="cuda")
    p2 = [ctypes.c_void_p(o2[i * 200:(i + 1) * 200].data_ptr()) for i in range(5)]
    rc = lib.fc_prepare(h, ctypes.c_void_p(big.data_ptr()), 8, 200, 0, *p2, None, ctypes.byref(info))
    assert rc == _lib.ERR_BATCH_EXCEEDS_CAPACITY and lib.fc_free_count(h) == 100
    assert lib.fc_prepare(h, None, 3, 1, 0, *p, None, ctypes.byref(info)) == _lib.ERR_BAD_ARG  # ids_bytes
    ok = torch.tensor([5, 5, 9], dtype=torch.int64, device="cuda")
    assert lib.fc_prepare(h, ctypes.c_void_p(ok.data_ptr()), 8, n, 0, *p, None, ctypes.byref(info)) == _lib.OK
    assert (info.unique, info.misses, lib.fc_free_count(h)) == (2, 2, 98)
    slots = torch.tensor([100], dtype=torch.int64, device="cuda")
    assert lib.fc_mark_dirty(h, ctypes.c_void_p(slots.data_ptr()), 1, None) == _lib.ERR_SLOT_OUT_OF_RANGE
    assert lib.fc_warmup(h, 5, None) == _lib.ERR_NOT_EMPTY
    lib.fc_destroy(h)


def test_pipeline_sequencing_rules():
    h, _ = make()
    assert lib.fc_set_engine(h, 1) == _lib.OK
    n = 4
    ids = torch.tensor([1, 2, 3, 4], dtype=torch.int64, device="cuda")
    out = torch.empty(10 * n, dtype=torch.int32, device="cuda")
    p = [ctypes.c_void_p(out[i * n:(i + 1) * n].data_ptr()) for i in range(5)]
    p2 = [ctypes.c_void_p(out[i * n:(i + 1) * n].data_ptr()) for i in range(5, 10)]
    info = _lib.PrepareInfo()
    assert lib.fc_prepare_commit(h, None, ctypes.byref(info)) == _lib.ERR_BAD_ARG  # nothing to commit
    assert lib.fc_prepare_begin(h, ctypes.c_void_p(ids.data_ptr()), 8, n, 0, *p, None) == _lib.OK
    assert lib.fc_prepare_begin(h, ctypes.c_void_p(ids.data_ptr()), 8, n, 1, *p2, None) == _lib.OK  # depth 2
    assert lib.fc_prepare_begin(h, ctypes.c_void_p(ids.data_ptr()), 8, n, 2, *p, None) == _lib.ERR_BAD_ARG
    assert b"outstanding" in lib.fc_last_error()
    rows = ctypes.c_int64()
    assert lib.fc_flush(h, None, ctypes.byref(rows)) == _lib.ERR_BAD_ARG       # sync verbs wait for the commits
    assert lib.fc_set_engine(h, 0) == _lib.ERR_BAD_ARG
    assert lib.fc_set_modes(h, 1, 0) == _lib.ERR_BAD_ARG                        # a mode change too
    assert lib.fc_set_modes(h, 0, 0) == _lib.OK                                 # the same modes are fine
    assert lib.fc_prepare(h, ctypes.c_void_p(ids.data_ptr()), 8, n, 0, *p, None, ctypes.byref(info)) == _lib.ERR_BAD_ARG
    assert lib.fc_prepare_commit(h, None, ctypes.byref(info)) == _lib.OK       # FIFO: batch 0 first
    assert (info.unique, info.misses, info.rows_to_slow) == (4, 4, -1)
    assert lib.fc_flush(h, None, ctypes.byref(rows)) == _lib.ERR_BAD_ARG       # batch 1 still outstanding
    assert lib.fc_prepare_commit(h, None, ctypes.byref(info)) == _lib.OK
    assert (info.unique, info.misses, info.hits) == (4, 0, 4)
    wb = ctypes.c_int64()
    assert lib.fc_last_writebacks(h, ctypes.byref(wb)) == _lib.OK and wb.value == 0
    assert lib.fc_flush(h, None, ctypes.byref(rows)) == _lib.OK and rows.value == 0
    # a zero-copy engine cannot prefetch
    assert lib.fc_set_engine(h, 0) == _lib.OK
    assert lib.fc_prepare_begin(h, ctypes.c_void_p(ids.data_ptr()), 8, n, 2, *p, None) == _lib.ERR_BAD_ARG
    lib.fc_destroy(h)
