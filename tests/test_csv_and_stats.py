"""CPU: trace ingestion (workload.load_csv / save_csv, workload.py:276-392) and the FQTB
statistics file (freq_stats.py:171-199) against outputs recorded from the REAL reference
(tests/golden/make_golden.py gen_csv): the reference's own load_csv test shapes, a
categorical log with string tokens, quoted fields and blank values, and the byte format
of save_csv."""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN

from paper_2208_05321_b200 import freq_stats, workload

DOC = json.load(open(os.path.join(GOLDEN, "csv.json")))


@pytest.mark.parametrize("name", sorted(DOC["load_csv"]))
def test_load_csv_matches_reference(name, tmp_path):
    case = DOC["load_csv"][name]
    path = tmp_path / (name + ".csv")
    with open(path, "w", newline="") as fh:
        fh.write(case["text"])
    if "error" in case:
        with pytest.raises(ValueError) as ei:
            workload.load_csv(path, **case["kwargs"])
        assert str(ei.value).replace(str(path), "<path>") == case["error"]
        return
    tr = workload.load_csv(path, **case["kwargs"])
    assert tr.num_ids == case["num_ids"] and tr.features == case["features"]
    assert tr.table_sizes == case["table_sizes"]
    assert np.array_equal(tr.samples, np.asarray(case["samples"], dtype=np.int64).reshape(-1, tr.features))


def test_column_remap_carries_across_files(tmp_path):
    """A ColumnRemap built on one file keeps ids stable on the next (new tokens appended)."""
    a, b = tmp_path / "a.csv", tmp_path / "b.csv"
    a.write_text("f0,f1\nx,y\nz,y\n")
    b.write_text("f0,f1\nz,w\nq,y\n")
    t1 = workload.load_csv(a)
    remap = workload.ColumnRemap(maps=[{"x": 0, "z": 1}, {"y": 0}], offsets=np.zeros(2, np.int64), num_ids=0)
    t2 = workload.load_csv(b, id_remap=remap)
    assert t1.table_sizes == [2, 1] and t2.table_sizes == [3, 2]
    assert t2.samples.tolist() == [[1, 3 + 1], [2, 3 + 0]]


def test_save_csv_bytes_match_reference(tmp_path):
    samples = np.asarray(DOC["trace_global_samples"], dtype=np.int64)
    tr = workload.Trace(3000, samples.shape[1], samples)
    path = tmp_path / "t.csv"
    workload.save_csv(tr, path)
    assert path.read_bytes() == open(os.path.join(GOLDEN, "trace_global.csv"), "rb").read()
    back = workload.load_csv(path, id_remap="identity", num_ids=3000)
    assert np.array_equal(back.samples, samples)


def test_fqtb_statistics_file_roundtrip(tmp_path):
    """save_table / load_table (freq_stats.py:171-199): counts survive, garbage and a
    corrupted checksum are refused; the reorder built from the loaded table is the same."""
    tr = workload.gen_zipf(300, 1.4, 900, 2, seed=9)
    table = freq_stats.scan_frequencies(tr.samples, 300)
    path = tmp_path / "stats.bin"
    freq_stats.save_table(table, path)
    raw = path.read_bytes()
    assert raw[:4] == b"FQTB" and len(raw) == 32 + 16 * int(np.count_nonzero(table.counts))
    loaded = freq_stats.load_table(path)
    assert loaded.num_ids == table.num_ids and np.array_equal(loaded.counts, table.counts)
    assert np.array_equal(freq_stats.build_reorder(loaded).rank_of, freq_stats.build_reorder(table).rank_of)
    (tmp_path / "junk.bin").write_bytes(b"not a stats file at all.....")
    with pytest.raises(ValueError):
        freq_stats.load_table(tmp_path / "junk.bin")
    bad = bytearray(raw)
    bad[-1] ^= 0x01  # one count changed: the header's total no longer matches
    (tmp_path / "bad.bin").write_bytes(bytes(bad))
    with pytest.raises(ValueError, match="checksum"):
        freq_stats.load_table(tmp_path / "bad.bin")
    j = freq_stats.table_from_json(freq_stats.table_to_json(table))
    assert np.array_equal(j.counts, table.counts)
