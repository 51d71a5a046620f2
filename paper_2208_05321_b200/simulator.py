"""`run(SimConfig)` on the GPU cache: the reference simulator's per-batch loop
(/root/reference/pkg/src/freqcache/simulator.py:353-528) driving the device
`CacheStack`s, emitting the same `RunMetrics` document (per-batch series, summary,
per-shard tallies; simulator.py:263-296) so the reference's metrics tooling and
`replay_eviction_law` consume GPU runs unchanged.

Supported: static-frequency LFU (`freq_lfu`) and its row-wise transfer accounting
(`rowwise_transfer`), column sharding (`num_shards` private caches over column
slices, sharding.py:62-118), synthetic traces (presets or explicit Zipf law),
both write-back and eviction modes, the dense oracle check (`track_oracle`) and the
event log. The runtime-LFU / LRU comparison baselines, CSV traces and table-wise
placement statistics are experiment tooling outside the hot path.
Optional (not in the reference): `prefetch=True` runs every shard through the
prefetch pipeline; the metrics are identical.

The GPU wall-clock per phase is reported under `gpu_timing`, which — like
`created_unix` / `elapsed_s` — is left out of `determinism_json`.
"""

from __future__ import annotations

import json
import time
from dataclasses import asdict, dataclass, replace

import numpy as np

from . import workload
from .freq_stats import build_reorder, scan_frequencies
from .sharding import build_column_stacks, partition_columns
from .store import fast_capacity
from .transmitter import DEFAULT_BUFFER_BYTES, ChannelModel, TransferReport
from .updates import update_column_weights, update_row_scalars

TOOL_VERSION = "0.1.0"
TRACE_FORMATS = ("global", "categorical")
POLICIES = ("freq_lfu", "rowwise_transfer")
NONDETERMINISTIC_FIELDS = ("created_unix", "elapsed_s", "gpu_timing")
TO_FAST = "to_fast"


@dataclass
class SimConfig:
    """The reference's SimConfig (simulator.py:120-197), GPU-backed subset."""

    preset: str | None = "criteo_like"
    exponent: float | None = None
    shift: float = 0.0
    trace_path: str | None = None
    trace_format: str = "global"
    num_ids: int = 1_000_000
    features: int | None = None
    num_batches: int = 100
    batch_size: int = 16384
    embedding_dim: int = 128
    cache_ratio: float = 0.015
    policy: str = "freq_lfu"
    write_back: str = "dirty_only"
    evict_mode: str = "occupancy_aware"
    shard_strategy: str = "column"
    num_shards: int = 1
    buffer_bytes: int = DEFAULT_BUFFER_BYTES
    latency_s: float = ChannelModel().latency_s
    bandwidth_Bps: float = ChannelModel().bandwidth_Bps
    local_bandwidth_Bps: float = ChannelModel().local_bandwidth_Bps
    seed: int = 0
    track_oracle: bool = False
    log_events: bool = False
    table_sizes: list | None = None

    def validate(self) -> None:
        if self.policy not in POLICIES:
            raise NotImplementedError(f"policy {self.policy!r} is a comparison baseline outside the GPU path; "
                                      f"have {POLICIES}")
        if self.shard_strategy != "column":
            raise NotImplementedError("table-wise placement statistics are not on the GPU path")
        if self.trace_format not in TRACE_FORMATS:
            raise ValueError(f"trace_format must be one of {TRACE_FORMATS}")
        if self.write_back not in ("dirty_only", "always"):
            raise ValueError(f"write_back must be 'dirty_only' or 'always', got {self.write_back!r}")
        if self.evict_mode not in ("occupancy_aware", "paper_literal"):
            raise ValueError("evict_mode must be 'occupancy_aware' or 'paper_literal'")
        if not (0.0 < self.cache_ratio <= 1.0):
            raise ValueError(f"cache_ratio must be in (0, 1], got {self.cache_ratio}")
        if self.num_ids < 1 or self.embedding_dim < 1:
            raise ValueError("num_ids and embedding_dim must be >= 1")
        if self.batch_size < 1 or self.num_batches < 0:
            raise ValueError("batch_size must be >= 1 and num_batches >= 0")
        if self.num_shards < 1:
            raise ValueError("num_shards must be >= 1")
        if self.trace_path is None and self.preset is None and self.exponent is None:
            raise ValueError("need a trace source: preset, exponent, or trace_path")
        if self.trace_path is None and self.preset is not None and self.preset not in workload.PRESETS:
            raise ValueError(f"unknown preset {self.preset!r}, have {sorted(workload.PRESETS)}")

    def channel(self) -> ChannelModel:
        return ChannelModel(self.latency_s, self.bandwidth_Bps, self.local_bandwidth_Bps)

    def resolved(self) -> dict:
        doc = asdict(self)
        doc["capacity"] = fast_capacity(self.num_ids, self.cache_ratio)
        if self.trace_path is not None:  # a CSV trace: nothing generated, nothing resolved (simulator.py:185)
            return doc
        if self.preset is not None:
            exp, shift = workload.preset_params(self.preset, self.num_ids)
            doc["exponent_resolved"] = exp
            doc["shift_resolved"] = shift
            doc["features_resolved"] = self.features if self.features is not None else \
                workload.PRESETS[self.preset].features
        else:
            doc["exponent_resolved"] = self.exponent
            doc["shift_resolved"] = self.shift
            doc["features_resolved"] = self.features if self.features is not None else 1
        return doc


def derive_seeds(seed: int) -> dict:
    """Independent named substreams (simulator.py:200-205)."""
    children = np.random.SeedSequence(seed).spawn(3)
    return {n: int(c.generate_state(1, np.uint64)[0]) for n, c in zip(("trace", "init", "updates"), children)}


def build_trace(config: SimConfig) -> workload.Trace:
    """The run's trace (simulator.py:208-225): a CSV file (global ids, or categorical columns
    remapped with per-feature offsets) or a generated stream."""
    if config.trace_path is not None:
        if config.trace_format == "global":
            return workload.load_csv(config.trace_path, id_remap="identity", num_ids=config.num_ids)
        return workload.load_csv(config.trace_path)
    seeds = derive_seeds(config.seed)
    n = config.num_batches * config.batch_size
    if config.preset is not None:
        return workload.gen_preset(config.preset, config.num_ids, n, seeds["trace"], features=config.features)
    return workload.gen_zipf(config.num_ids, config.exponent, n, config.features if config.features else 1,
                             seeds["trace"], shift=config.shift)


@dataclass
class RunMetrics:
    """The reference's metrics document (simulator.py:263-296)."""

    config: dict
    per_batch: dict
    summary: dict
    per_shard: list
    tool_version: str = TOOL_VERSION
    created_unix: float = 0.0
    elapsed_s: float = 0.0
    gpu_timing: dict | None = None

    def to_dict(self) -> dict:
        return {"schema_version": 1, "tool_version": self.tool_version, "created_unix": self.created_unix,
                "elapsed_s": self.elapsed_s, "config": self.config, "per_batch": self.per_batch,
                "summary": self.summary, "per_shard": self.per_shard, "gpu_timing": self.gpu_timing}

    def to_json(self, indent: int | None = 2) -> str:
        return json.dumps(self.to_dict(), indent=indent, sort_keys=True)

    def determinism_json(self) -> str:
        doc = self.to_dict()
        for key in NONDETERMINISTIC_FIELDS:
            doc.pop(key, None)
        return json.dumps(doc, sort_keys=True)


def _empty_tally() -> dict:
    return {"rows_to_fast": 0, "bytes_to_fast": 0, "messages_to_fast": 0, "rows_to_slow": 0, "bytes_to_slow": 0,
            "messages_to_slow": 0, "modeled_time_s": 0.0}


def _tally(t: dict, reports) -> None:
    for rep in reports:
        side = "to_fast" if rep.direction == TO_FAST else "to_slow"
        t[f"rows_{side}"] += rep.rows
        t[f"bytes_{side}"] += rep.bytes
        t[f"messages_{side}"] += rep.messages
        t["modeled_time_s"] += rep.modeled_time_s


def _run_stacks(config: SimConfig, trace: workload.Trace | None, prefetch: bool = False, device=None):
    import torch

    t0 = time.perf_counter()
    config.validate()
    if trace is None:
        trace = build_trace(config)
    if trace.num_ids != config.num_ids:
        config = replace(config, num_ids=trace.num_ids)
    seeds = derive_seeds(config.seed)
    idx_map = build_reorder(scan_frequencies(trace, config.num_ids))
    plan = partition_columns(config.embedding_dim, config.num_shards)
    mode = "rowwise" if config.policy == "rowwise_transfer" else "block"
    stacks = build_column_stacks(idx_map, plan, config.embedding_dim, config.cache_ratio, seeds["init"],
                                 channel=config.channel(), buffer_bytes=config.buffer_bytes, transmitter_mode=mode,
                                 write_back=config.write_back, evict_mode=config.evict_mode,
                                 log_events=config.log_events, with_reference=config.track_oracle, device=device,
                                 engine="async")
    capacity = stacks[0].capacity
    shard_t = [{"warmup": _empty_tally(), "batch_phase": _empty_tally(), "flush": _empty_tally()} for _ in stacks]
    warm_t = _empty_tally()
    tw = time.perf_counter()
    for i, st in enumerate(stacks):
        rep = st.warmup(capacity)
        _tally(warm_t, [rep])
        _tally(shard_t[i]["warmup"], [rep])
    torch.cuda.synchronize()
    t_warm = time.perf_counter() - tw

    col_w = update_column_weights(config.embedding_dim, seeds["updates"])
    keys = ("unique", "hits", "misses", "evictions", "hit_ratio", "bytes_to_fast", "bytes_to_slow", "rows_to_fast",
            "rows_to_slow", "messages", "modeled_transfer_time_s")
    per_batch = {k: [] for k in keys}
    batch_t = _empty_tally()
    counters = {"prepare_calls": 0, "ids_processed": 0, "unique_ids_processed": 0}
    batches = list(workload.batches(trace, config.batch_size))
    tb = time.perf_counter()
    nxt = None
    for i, batch in enumerate(batches):
        try:
            preps = [st.prepare(batch.ids, batch.seq) for st in stacks]
        except Exception as exc:
            raise type(exc)(f"batch {batch.seq}: {exc}") from exc
        p0 = preps[0]
        for p in preps[1:]:  # column shards decide identically (simulator.py:422-426)
            assert (p.hits, p.misses, p.evictions) == (p0.hits, p0.misses, p0.evictions)
        if prefetch and i + 1 < len(batches):
            nxt = batches[i + 1]
            for st in stacks:
                st.prefetch(nxt.ids, nxt.seq)
        if p0.num_unique:
            for st, prep in zip(stacks, preps):
                _ = st.gather_unique(prep)  # the simulated lookup
                st.apply_synthetic_update(prep, batch.seq, seeds["updates"], col_w)
        step = _empty_tally()
        for s, prep in enumerate(preps):
            _tally(step, prep.transfer_reports)
            _tally(shard_t[s]["batch_phase"], prep.transfer_reports)
            counters["prepare_calls"] += 1
        counters["ids_processed"] += int(batch.ids.size)
        counters["unique_ids_processed"] += int(p0.num_unique)
        per_batch["unique"].append(int(p0.num_unique))
        per_batch["hits"].append(int(p0.hits))
        per_batch["misses"].append(int(p0.misses))
        per_batch["evictions"].append(int(p0.evictions))
        per_batch["hit_ratio"].append(p0.hits / max(1, p0.num_unique))
        for k in ("bytes_to_fast", "bytes_to_slow", "rows_to_fast", "rows_to_slow"):
            per_batch[k].append(step[k])
        per_batch["messages"].append(step["messages_to_fast"] + step["messages_to_slow"])
        per_batch["modeled_transfer_time_s"].append(step["modeled_time_s"])
        for k in batch_t:
            batch_t[k] += step[k]
    torch.cuda.synchronize()
    t_batches = time.perf_counter() - tb

    flush_t = _empty_tally()
    tf = time.perf_counter()
    for i, st in enumerate(stacks):
        rep = st.flush()
        _tally(flush_t, [rep])
        _tally(shard_t[i]["flush"], [rep])
    torch.cuda.synchronize()
    t_flush = time.perf_counter() - tf

    oracle = {"checked": bool(config.track_oracle), "ok": None, "first_divergence": None}
    if config.track_oracle:
        div = None
        for st in stacks:
            div = st.first_divergence()
            if div is not None:
                break
        oracle["ok"] = div is None
        oracle["first_divergence"] = div

    n_b = len(batches)
    steady = n_b // 10
    hits, uniq = sum(per_batch["hits"]), sum(per_batch["unique"])
    per_shard = [{"shard": i, "col_range": list(st.col_range), **st.memory_report(), **shard_t[i]}
                 for i, st in enumerate(stacks)]
    summary = {
        "batches": n_b, "capacity": capacity, "unique_refs": uniq, "hits": hits,
        "misses": sum(per_batch["misses"]), "evictions": sum(per_batch["evictions"]),
        "hit_ratio": hits / max(1, uniq),
        "steady_state_hit_ratio": sum(per_batch["hits"][steady:]) / max(1, sum(per_batch["unique"][steady:])),
        "steady_state_from_batch": steady, "warmup": warm_t, "batch_phase": batch_t, "flush": flush_t,
        "total_modeled_transfer_time_s": warm_t["modeled_time_s"] + batch_t["modeled_time_s"]
        + flush_t["modeled_time_s"],
        "peak_fast_tier_bytes": {
            "fast_rows_bytes": sum(s["fast_rows_bytes"] for s in per_shard),
            "buffer_bytes": sum(s["buffer_bytes"] for s in per_shard),
            "index_bytes": sum(s["index_bytes"] for s in per_shard),
            "total": sum(s["peak_fast_tier_bytes"] for s in per_shard)},
        "fast_row_fraction_of_full_residency": capacity / config.num_ids,
        "overhead_counters": counters,
        "oracle": oracle,
    }
    gpu = {"warmup_s": t_warm, "batches_s": t_batches, "flush_s": t_flush,
           "lookups_per_s": counters["ids_processed"] / max(t_batches, 1e-12), "prefetch": bool(prefetch)}
    metrics = RunMetrics(config=config.resolved(), per_batch=per_batch, summary=summary, per_shard=per_shard,
                         created_unix=time.time(), elapsed_s=time.perf_counter() - t0, gpu_timing=gpu)
    return metrics, stacks


def run(config: SimConfig, trace: workload.Trace | None = None, prefetch: bool = False, device=None) -> RunMetrics:
    """Simulate the whole trace on the GPU cache (simulator.py:525-528)."""
    metrics, _ = _run_stacks(config, trace, prefetch=prefetch, device=device)
    return metrics


def replay_eviction_law(events: list, num_ids: int) -> list:
    """Re-derive every eviction of a GPU run from its event log (simulator.py:571-621,
    static-frequency policies): the evicted set must be the `needed` largest occupied,
    unprotected ranks, and a protected rank is never evicted. Returns the violations."""
    if not events:
        return []
    if events[0].policy not in POLICIES:
        raise ValueError(f"cannot replay policy {events[0].policy!r} on the GPU path")
    occupied = np.zeros(num_ids, dtype=bool)
    violations = []
    for i, ev in enumerate(events):
        ev_r = np.asarray(ev.evicted_ranks, dtype=np.int64)
        if ev_r.size:
            prot = np.asarray(ev.protected_ranks, dtype=np.int64)
            if np.isin(ev_r, prot).any():
                violations.append({"event": i, "kind": "protected_evicted"})
            cand = np.flatnonzero(occupied)
            cand = cand[~np.isin(cand, prot)]
            expect = np.sort(cand)[-ev_r.size:]
            if not np.array_equal(expect, np.sort(ev_r)):
                violations.append({"event": i, "kind": "wrong_victims", "expected": expect.tolist(),
                                   "got": np.sort(ev_r).tolist()})
            occupied[ev_r] = False
        occupied[np.asarray(ev.admitted_ranks, dtype=np.int64)] = True
    return violations
