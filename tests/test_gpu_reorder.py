"""GPU frequency reorder (fc_build_reorder) against the reference's semantics:
scan_frequencies + build_reorder (/root/reference/pkg/src/freqcache/freq_stats.py:97-148),
pinned by the reference test's known answer (test_freq_stats.py:95-107) and, bit-exact,
by the numpy oracle on random traces with many ties."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle  # noqa: E402

pytestmark = pytest.mark.gpu

import paper_2208_05321_b200 as fc  # noqa: E402


def test_known_answer():
    # counts {5:3, 2:2, 9:1} over 10 ids -> rank_of[5,2,9] = 0,1,2; unseen ids follow in ascending order
    trace = np.array([5, 5, 5, 2, 2, 9])
    freq, idx = fc.build_reorder_device(trace, 10)
    assert idx.rank_of[[5, 2, 9]].tolist() == [0, 1, 2]
    assert idx.id_of[3:].tolist() == [0, 1, 3, 4, 6, 7, 8]
    assert freq.counts.tolist() == np.bincount(trace, minlength=10).tolist()
    # uniform counts -> identity
    _, idx = fc.build_reorder_device(np.arange(50), 50)
    assert np.array_equal(idx.rank_of, np.arange(50))


@pytest.mark.parametrize("num_ids,n,alpha,dtype", [(1000, 5000, 1.05, np.int64), (200_000, 2_000_000, 1.05, np.int32),
                                                   (70_001, 300_000, 0.6, np.int64), (5, 1, 1.0, np.int32)])
def test_matches_oracle(num_ids, n, alpha, dtype):
    rng = np.random.default_rng(num_ids)
    p = 1.0 / np.arange(1, num_ids + 1) ** alpha
    trace = rng.permutation(num_ids)[rng.choice(num_ids, size=n, p=p / p.sum())].astype(dtype)
    freq, idx = fc.build_reorder_device(trace, num_ids)
    counts = oracle.frequency_counts(trace, num_ids)
    rank_of, id_of = oracle.rank_permutation(counts)
    assert np.array_equal(freq.counts, counts)
    assert np.array_equal(idx.id_of, id_of) and np.array_equal(idx.rank_of, rank_of)
    idx.check()
    # and through the package's CPU restatement
    ref = fc.build_reorder(fc.scan_frequencies(trace, num_ids))
    assert np.array_equal(ref.rank_of, idx.rank_of)


def test_device_tensor_input_and_errors():
    t = torch.tensor([3, 1, 3, 0], device="cuda")
    _, idx = fc.build_reorder_device(t, 4)
    assert idx.id_of.tolist() == [3, 0, 1, 2]
    with pytest.raises(ValueError, match="-2"):
        fc.build_reorder_device(np.array([1, -2, 7, -1]), 5)
    with pytest.raises(ValueError, match="9"):
        fc.build_reorder_device(np.array([1, 9, 7]), 5)
    _, idx = fc.build_reorder_device(np.empty(0, np.int64), 3)
    assert idx.id_of.tolist() == [0, 1, 2]
