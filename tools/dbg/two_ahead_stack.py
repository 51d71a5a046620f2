import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import oracle
import paper_2208_05321_b200 as fc

rng = np.random.default_rng(21)
num_ids, dim, steps, B = 6_000, 8, 6, 2_000
p = 1.0 / np.arange(1, num_ids + 1) ** 0.9
trace = rng.permutation(num_ids)[rng.choice(num_ids, size=(steps, B), p=p / p.sum())]
rank_of, id_of = oracle.rank_permutation(oracle.frequency_counts(trace, num_ids))
ref = oracle.init_rows(num_ids, dim, 1)
cap = 1500
deltas = [rng.standard_normal((B, dim)).astype(np.float32) for _ in range(steps)]

def run(pattern):
    orc = oracle.OracleCache(rank_of, ref[id_of].copy(), cap)
    st = fc.CacheStack(fc.IdxMap(rank_of, id_of), fc.SlowTierStore(ref[id_of].copy()),
                       fc.FastTierStore(np.zeros((cap, dim), np.float32)), fc.Transmitter(), log_events=True,
                       engine="async")
    b = [trace[s] for s in range(steps)]
    if pattern == "ahead":
        st.prefetch(b[0], 0); st.prefetch(b[1], 1)
    for s in range(steps):
        if pattern == "depth2":
            if s == 0: st.prefetch(b[0], 0)
            if s + 1 < steps: st.prefetch(b[1 + s], s + 1)
        q = st.prepare(b[s], s)
        a = orc.prepare(b[s], s)
        if pattern == "ahead" and s + 2 < steps:
            st.prefetch(b[s + 2], s + 2)
        ok = (q.hits, q.misses, q.evictions) == (a["hits"], a["misses"], a["evictions"]) and \
            np.array_equal(q.unique_slots, a["unique_slots"]) and np.array_equal(st.events[-1].evicted_ranks, a["evicted"])
        torch.cuda.synchronize()
        fr = st.fast.slots.cpu().numpy()
        occ = orc.slot_rank >= 0
        rows_ok = np.array_equal(fr[occ], orc.fast[occ]) if hasattr(orc, "fast") else None
        print(pattern, s, "decisions", ok, "fast rows", rows_ok, flush=True)
        st.scatter_update(q, deltas[s])
        orc.scatter_update(a, deltas[s])
    st.flush(); orc.flush(); torch.cuda.synchronize()
    print(pattern, "slow tier equal", np.array_equal(st.slow.rows, orc.slow))

for pat in ("none", "depth2", "ahead"):
    run(pat)
