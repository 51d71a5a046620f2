"""Table-wise sharding host logic (CPU): the reference's placement and load statistics
(plan_tables_greedy / tablewise_imbalance / columnwise_imbalance, sharding.py:149-205)
against golden values recorded from the reference (tests/golden/tablewise.json, made by
make_golden.py gen_tablewise), and TablePlacement's owner/owner-local map — the map
fc_router_create_tables' kernels implement (test_gpu_router checks the two agree)."""

import json
import os

import numpy as np
import pytest
import torch

import paper_2208_05321_b200 as fc
from paper_2208_05321_b200.distributed import TablePlacement

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "tablewise.json")))


@pytest.mark.parametrize("key", sorted(k for k in GOLD if not k.startswith("column/")))
def test_plan_tables_greedy_matches_reference(key):
    g = GOLD[key]
    w = int(key.split("/")[1])
    plan = fc.plan_tables_greedy(g["sizes"], w)
    assert plan.assignment.tolist() == g["assignment"]
    st = fc.tablewise_imbalance(plan)
    assert st.per_shard_rows.tolist() == g["per_shard_rows"] and st.max_rows == g["max_rows"]
    assert st.mean_rows == g["mean_rows"] and st.imbalance_ratio == g["imbalance_ratio"]


@pytest.mark.parametrize("key", sorted(k for k in GOLD if k.startswith("column/")))
def test_columnwise_imbalance_matches_reference(key):
    _, dim, w = key.split("/")
    st = fc.columnwise_imbalance(fc.partition_columns(int(dim), int(w)), 33_762_577)
    g = GOLD[key]
    assert st.per_shard_rows.tolist() == g["per_shard_rows"] and st.imbalance_ratio == g["imbalance_ratio"]


def test_plan_rejects_bad_input():
    with pytest.raises(ValueError):
        fc.plan_tables_greedy([], 2)
    with pytest.raises(ValueError):
        fc.plan_tables_greedy([3, 4], 0)


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_table_placement_maps_every_id_once(world):
    """Criteo's 26 tables scaled down: every global id maps to exactly one (owner, local)
    pair, each owner's local ids are 0..rows-1 with its tables in table order, and
    global_ids inverts the map."""
    sizes = fc.criteo_like_table_sizes(1000)
    pl = TablePlacement.balanced(sizes, world)
    assert pl.owner.tolist() == GOLD[f"criteo_div1000/{world}"]["assignment"]
    ids = torch.arange(pl.num_ids)
    own, loc = pl.owner_local(ids)
    for r in range(world):
        mine = loc[own == r].numpy()
        assert np.array_equal(np.sort(mine), np.arange(pl.local_sizes[r]))
        g = pl.global_ids(r)
        assert g.size == pl.local_sizes[r]
        o2, l2 = pl.owner_local(torch.from_numpy(g))
        assert (o2 == r).all() and np.array_equal(l2.numpy(), np.arange(g.size))
        # tables in table order inside an owner
        tabs = [t for t in range(len(sizes)) if pl.owner[t] == r]
        assert [int(pl.lbase[t]) for t in tabs] == list(np.concatenate([[0], np.cumsum([sizes[t] for t in tabs])])[:-1])


def test_table_placement_rejects_bad_layouts():
    with pytest.raises(ValueError):
        TablePlacement([0, 5, 5, 9], [0, 1, 0], 2)  # empty table
    with pytest.raises(ValueError):
        TablePlacement([0, 5, 9], [0, 2], 2)  # owner outside the world
    with pytest.raises(ValueError):
        TablePlacement([1, 5, 9], [0, 1], 2)  # does not start at 0
