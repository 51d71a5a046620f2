"""CPU (no GPU): the C-ABI library loads and exports every symbol the header
declares; host-side logic (transfer accounting, column plan, update hash, reorder)
matches the oracle. No compute calls into the library here."""

import ctypes
import os
import re

import numpy as np
import pytest

import oracle
from conftest import ROOT

import paper_2208_05321_b200 as fc
from paper_2208_05321_b200 import _lib, updates

HEADER = os.path.join(ROOT, "include", "freqcache_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|const char\*)\s+(fc_\w+)\s*\(", text, re.M)))


def test_library_exports_every_header_symbol():
    if not os.path.exists(_lib.LIB_PATH):
        from paper_2208_05321_b200 import build

        build.build(verbose=False)
    lib = ctypes.CDLL(_lib.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_lib.EXPORTS)
    _lib.load()  # argtypes bind


def test_library_is_sm100a():
    out = os.popen(f"cuobjdump --list-elf {_lib.LIB_PATH} 2>/dev/null").read()
    if not out:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out


def test_chunk_plan_and_reports():
    MiB = 2**20
    assert fc.chunk_plan(0, 512, MiB) == 0
    assert fc.chunk_plan(16384, 512, 64 * MiB) == 1
    assert fc.chunk_plan(16384, 512, MiB) == 8
    assert fc.chunk_plan(3, 400, 1000) == 2
    with pytest.raises(fc.BufferTooSmall):
        fc.chunk_plan(1, 2 * MiB, MiB)
    tx = fc.Transmitter(buffer=fc.TransferBuffer(MiB))
    r = tx.report("to_fast", 16384, 512)
    assert (r.rows, r.bytes, r.messages) == (16384, 16384 * 512, 8)
    ch = fc.ChannelModel()
    assert r.modeled_time_s == pytest.approx(ch.block_time_s(8, 16384 * 512))
    assert fc.Transmitter(mode="rowwise").report("to_slow", 10, 512).messages == 10
    with pytest.raises(ValueError):
        fc.ChannelModel(latency_s=0.0)
    for rows in range(0, 50):
        assert fc.chunk_plan(rows, 400, 1000) == oracle.chunk_messages(rows, 400, 1000)


def test_partition_columns_matches_oracle():
    assert fc.partition_columns(10, 3).ranges == ((0, 4), (4, 7), (7, 10))
    for dim in (1, 7, 10, 64, 128):
        for n in range(1, min(dim, 9) + 1):
            assert list(fc.partition_columns(dim, n).ranges) == oracle.column_ranges(dim, n)
    with pytest.raises(ValueError):
        fc.partition_columns(4, 5)
    rep = fc.alltoall_volume(16384, 128, 4)
    assert rep.per_pair_bytes == 524_288 and rep.total_bytes == 524_288 * 12


def test_update_hash_matches_oracle():
    rng = np.random.default_rng(0)
    ids = rng.integers(0, 2**40, 1000)
    cnt = rng.integers(1, 100, 1000)
    for seq, seed in ((0, 1), (99, 2**63 + 5), (12345, 7)):
        assert np.array_equal(updates.update_row_scalars(ids, cnt, seq, seed), oracle.row_scalars(ids, cnt, seq, seed))
    assert np.array_equal(updates.update_column_weights(128, 42), oracle.column_weights(128, 42))


def test_reorder_and_init_match_oracle():
    rng = np.random.default_rng(4)
    for n in (1, 5, 300, 4096):
        c = rng.integers(0, 4, n)
        m = fc.build_reorder(fc.FrequencyTable(counts=c, num_ids=n))
        r, i = oracle.rank_permutation(c)
        assert np.array_equal(m.rank_of, r) and np.array_equal(m.id_of, i)
        m.check()
    assert np.array_equal(fc.init_reference_rows(1000, 8, 123), oracle.init_rows(1000, 8, 123))
    assert fc.fast_capacity(1_000_000, 0.015) == 15_000
    with pytest.warns(UserWarning):
        assert fc.fast_capacity(100, 0.005) == 1


def test_cache_state_validation_without_gpu():
    with pytest.raises(ValueError):
        fc.CacheState(0, 10)
    with pytest.raises(ValueError):
        fc.CacheState(11, 10)
    st = fc.CacheState(4, 10)
    assert st.free_count == 4 and (st.slot_to_rank == -1).all()


def test_simulator_config_and_presets_match_reference_goldens():
    """The GPU simulator's host side (SimConfig.resolved, preset calibration) against the
    reference's recorded RunMetrics config (tests/golden/sim_metrics.json)."""
    import json

    from conftest import GOLDEN
    from paper_2208_05321_b200 import simulator

    docs = json.load(open(os.path.join(GOLDEN, "sim_metrics.json")))
    for doc in docs.values():
        cfg = simulator.SimConfig(**doc["config"])
        cfg.validate()
        assert cfg.resolved() == doc["metrics"]["config"]
    with pytest.raises(NotImplementedError):
        simulator.SimConfig(policy="lru").validate()


def test_peer_rows_bound_is_checked_on_the_full_count_matrix():
    """An owner writes into (and reads from) EVERY requester's peer buffer, so the buffer
    bound is checked against the largest row of the all-gathered count matrix before any
    peer kernel runs -- not only against this rank's own routed count."""
    import torch

    from paper_2208_05321_b200.distributed import PeerRows

    pr = object.__new__(PeerRows)
    pr.rank, pr.world, pr.max_rows, pr.device = 0, 2, 10, torch.device("cpu")
    x = {"mat": [[3, 4], [6, 6]], "rc": [3, 6], "u": 7}  # this rank routes 7 <= 10; rank 1 routes 12
    with pytest.raises(RuntimeError, match="routes 12"):
        pr.segments(x)
    x = {"mat": [[3, 4], [4, 6]], "rc": [3, 4], "u": 7}
    pr.segments(x)
    assert x["seg"].tolist() == [0, 3, 7] and x["off"].tolist() == [0, 0]


def test_bench_reference_arm_and_gpu_count_check():
    """bench.py's CPU arm prints one JSON line with the driver's keys (the reference package
    from baseline/_ref when installed, else the oracle port), and `--gpus N` on a host with
    fewer GPUs fails loudly instead of silently running one rank."""
    import json
    import subprocess
    import sys

    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "small",
                        "--steps", "2", "--warmup", "1", "--trace-batches", "12"],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1
    doc = json.loads(lines[0])
    assert doc["impl"] == "reference" and doc["unit"] == "lookups/s" and doc["value"] > 0
    assert doc["cpu_baseline"]["kind"] in ("reference", "port") and doc["cpu_baseline"]["cores"] == 1
    assert doc["config"]["workload"] == "small" and doc["config"]["parallelism"] == "single"
    assert doc["e2e"]["h2d_bytes_per_step"] == 0
    # rank 0 of a 2-rank launch: the config's batch is the global batch (strong scaling), split in
    # two, and the reference's column-wise stacks serve it
    env = dict(os.environ, WORLD_SIZE="2", RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "small",
                        "--gpus", "2", "--shard", "column", "--steps", "1", "--warmup", "3", "--trace-batches", "12"],
                       capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    doc = json.loads([ln for ln in r.stdout.splitlines() if ln.strip()][0])
    assert doc["scaling"] == "strong" and doc["n_gpus"] == 2
    assert doc["config"]["global_batch"] == 1024 and doc["config"]["batch_per_gpu"] == 512
    assert doc["config"]["parallelism"] == "columnwise2" and doc["config"]["lookups_per_step"] == 1024 * 26
    import torch

    if torch.cuda.device_count() < 2:
        r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1"],
                           capture_output=True, text=True, timeout=300)
        assert r.returncode != 0 and "CUDA device" in r.stderr
