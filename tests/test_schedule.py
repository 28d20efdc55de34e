"""Host-side schedule mirror (paper_2305_18627_b200.gqsgd) vs the reference.

The tree / ring event lists are part of the exponential path's parity
contract (the k draws are keyed by (step, dst)); these are pure host logic,
so they are checked on CPU against the reference's own KATs
(proj/tests/test_topology.cpp) and against the compiled reference."""
import pytest

from paper_2305_18627_b200.gqsgd import (chunk_lane_range, make_schedule, ring_schedule,
                                         tree_schedule, TopologyKind)


def events(s):
    return [(e.step, e.src, e.dst, e.op, e.chunk) for e in s.events]


def test_tree5_events():  # test_topology.cpp:76-97
    want = [(0, 1, 0, 0, 0), (0, 3, 2, 0, 0), (1, 2, 0, 0, 0), (2, 4, 0, 0, 0),
            (3, 0, 4, 1, 0), (4, 0, 2, 1, 0), (5, 0, 1, 1, 0), (5, 2, 3, 1, 0)]
    s = tree_schedule(5)
    assert events(s) == want and s.steps == 6 and s.chunks == 1


def test_ring3_events():  # test_topology.cpp:125-146
    rs = [(0, 0, 1, 0, 0), (0, 1, 2, 0, 1), (0, 2, 0, 0, 2),
          (1, 0, 1, 0, 2), (1, 1, 2, 0, 0), (1, 2, 0, 0, 1)]
    s = ring_schedule(3)
    ev = events(s)
    assert ev[:6] == rs and all(e[3] == 1 for e in ev[6:]) and len(ev) == 12 and s.chunks == 3


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 7, 8, 9, 16, 33])
@pytest.mark.parametrize("topo", [0, 1])
def test_schedules_match_oracle_and_reference(oracle, reference, n, topo):
    s = make_schedule(TopologyKind(topo), n)
    assert events(s) == oracle.schedule(topo, n)
    if reference is not None:
        assert events(s) == reference.schedule(topo, n)


def test_step_conflict_freedom():  # test_topology.cpp:54-64
    for n in range(1, 20):
        for s in (tree_schedule(n), ring_schedule(n)):
            by_step = {}
            for e in s.events:
                by_step.setdefault(e.step, []).append(e)
            for evs in by_step.values():
                written = {(e.dst, e.chunk) for e in evs}
                assert not any((e.src, e.chunk) in written for e in evs)


def test_chunk_lane_range():  # topology.cpp:99-106
    assert [chunk_lane_range(10, 3, c) for c in range(3)] == [(0, 3), (3, 6), (6, 10)]
    assert chunk_lane_range(0, 4, 3) == (0, 0)
    with pytest.raises(ValueError):
        chunk_lane_range(10, 3, 3)
