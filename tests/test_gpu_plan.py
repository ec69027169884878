"""GPU dedup planner (``ht_gplan_build``): every set of the plan
computed on the device from raw (duplicated) chunk neighbour ids is
bit-identical with the reference's planner - pinned against the golden
digests the unmodified reference produced (tests/golden/make_golden.py)
and against the host planner on larger grids."""

import numpy as np
import pytest

import paper_2311_14898_b200 as H
from conftest import TOY_EDGES, TOY_OWNER, TOY_RANGES, load_json, random_set_instances
from digest import plan_digest

pytestmark = pytest.mark.gpu


def _digest(plan):
    return plan_digest(plan.m, plan.n, plan.neighbor_sets, plan.union_sets, plan.owned_sets,
                       plan.carry_sets, plan.load_sets, plan.fetch_sets, plan.nbr_carry_sets,
                       plan.layout.live_sets, plan.layout.slots, plan.layout.capacities,
                       (plan.volumes.v_ori, plan.volumes.v_p2p, plan.volumes.v_ru))


def _raw(nbrs, rng):
    """Shuffled, duplicated neighbour ids (what a chunk's edge list holds)."""
    out = []
    for row in nbrs:
        r = []
        for s in row:
            s = np.asarray(s, np.int64)
            x = np.concatenate([s, rng.choice(s, size=s.size)]) if s.size else s
            r.append(rng.permutation(x))
        out.append(r)
    return out


def test_toy_grid(golden_toy):
    src = np.array([e[0] for e in TOY_EDGES])
    dst = np.array([e[1] for e in TOY_EDGES])
    g = H.from_edges(src, dst, num_vertices=8)
    p = H.two_level_from_ranges(g, H.PartitionAssignment(owner=TOY_OWNER.copy(), m=3), TOY_RANGES)
    plan = H.plan_for_partition(p, device=0)
    assert _digest(plan) == golden_toy["digest"]
    assert plan.layout.capacities == [4, 4, 3]
    for mode, pred in golden_toy["predicted"].items():
        assert H.predicted_transfers(plan, mode) == pred


def test_random_set_instances(golden_sets):
    rng = np.random.default_rng(5)
    for (nbrs, owner), gold in zip(random_set_instances(), golden_sets):
        plan = H.build_plan_gpu(_raw(nbrs, rng), owner, device=0)
        assert _digest(plan) == gold["digest"]


def test_matches_host_planner_on_random_partitions():
    from conftest import random_graph, random_two_level
    rng = np.random.default_rng(11)
    for _ in range(12):
        g = random_graph(rng, num_vertices=int(rng.integers(50, 400)))
        m, n = int(rng.integers(1, 5)), int(rng.integers(1, 6))
        p = random_two_level(g, rng, m, min(n, max(1, g.num_vertices // max(m, 1) // 2)))
        a, b = H.plan_for_partition(p), H.plan_for_partition(p, device=0)
        assert _digest(a) == _digest(b)


def test_out_of_range_ids_raise():
    with pytest.raises(H.PlanError):
        H.build_plan_gpu([[np.array([9])]], np.zeros(3, dtype=np.int64), device=0)
    with pytest.raises(H.PlanError):
        H.build_plan_gpu([[np.array([1])]], np.array([0, 5], dtype=np.int64), device=0)


@pytest.mark.slow
def test_cfg1_reorganized_plan_matches_reference():
    gold = load_json("cfg1.json")
    ds = H.synth_dataset(H.SynthSpec(num_vertices=100_000, avg_degree=20.0, seed=0), 64, 16)
    a = H.partition_vertices(ds.graph, 4, seed=0)
    r = H.reorganize(H.split_chunks(ds.graph, a, 4))
    plan = H.plan_for_partition(r.partition, device=0)
    assert _digest(plan) == gold["plan_digest_reorg"]
    assert plan.layout.capacities == gold["caps"]
    assert (plan.volumes.v_ori, plan.volumes.v_p2p, plan.volumes.v_ru) == tuple(gold["volumes_reorg"])
    # m = 8, n = 8 against the host planner
    a8 = H.partition_vertices(ds.graph, 8, seed=0)
    p8 = H.reorganize(H.split_chunks(ds.graph, a8, 8)).partition
    assert _digest(H.plan_for_partition(p8, device=0)) == _digest(H.plan_for_partition(p8))
