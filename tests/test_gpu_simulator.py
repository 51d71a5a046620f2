"""simulator.run on the GPU cache reproduces the reference simulator's RunMetrics
document (simulator.py:263-296, 353-528) exactly — per-batch series, summary,
per-shard tallies, resolved config — for golden runs recorded from the reference
(tests/golden/make_golden.py gen_sim_metrics), with and without the prefetch
pipeline; and the GPU run's event log satisfies the eviction law (:571-621)."""

import json
import math
import os

import pytest

torch = pytest.importorskip("torch")

from conftest import GOLDEN  # noqa: E402

pytestmark = pytest.mark.gpu

from paper_2208_05321_b200 import simulator  # noqa: E402

DOCS = json.load(open(os.path.join(GOLDEN, "sim_metrics.json")))


def close(a, b, path="doc"):
    if isinstance(a, dict):
        assert set(a) == set(b), (path, set(a) ^ set(b))
        for k in a:
            close(a[k], b[k], f"{path}.{k}")
    elif isinstance(a, list):
        assert len(a) == len(b), path
        for i, (x, y) in enumerate(zip(a, b)):
            close(x, y, f"{path}[{i}]")
    elif isinstance(a, float) or isinstance(b, float):
        assert math.isclose(a, b, rel_tol=1e-12, abs_tol=1e-18), (path, a, b)
    else:
        assert a == b, (path, a, b)


@pytest.mark.parametrize("name", sorted(DOCS))
@pytest.mark.parametrize("prefetch", [False, True])
def test_run_matches_reference_metrics(name, prefetch):
    doc = DOCS[name]
    cfg = simulator.SimConfig(**doc["config"])
    m = simulator.run(cfg, prefetch=prefetch)
    got = json.loads(m.determinism_json())
    close(got, doc["metrics"])
    assert m.gpu_timing["batches_s"] > 0


def test_event_log_obeys_eviction_law():
    cfg = simulator.SimConfig(**DOCS["preset_2shards_oracle"]["config"])
    metrics, stacks = simulator._run_stacks(cfg, None, prefetch=True)
    for st in stacks:
        assert st.events and simulator.replay_eviction_law(st.events, cfg.num_ids) == []
    assert metrics.summary["oracle"]["ok"] is True


CSV = json.load(open(os.path.join(GOLDEN, "csv.json")))


@pytest.mark.parametrize("name", sorted(CSV["runs"]))
def test_csv_trace_run_matches_reference_metrics(name, monkeypatch):
    """simulator.run on a CSV trace (simulator.py:208-213): save_csv's global-id format and a
    categorical log remapped with per-feature offsets (load_csv), fed to the device caches;
    the RunMetrics document equals the reference's."""
    from conftest import ROOT

    monkeypatch.chdir(ROOT)  # the recorded configs name the trace relative to the repo root
    doc = CSV["runs"][name]
    m = simulator.run(simulator.SimConfig(**doc["config"]), prefetch=True)
    close(json.loads(m.determinism_json()), doc["metrics"])
