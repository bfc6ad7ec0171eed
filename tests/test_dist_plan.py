"""The multi-rank decomposition and its halo / gather schedule, checked on CPU
with gloo at world sizes 2, 3, 4 and 8 (requirement (1) of
P:39-40, WRF-style horizontal patches).

Every rank asks the library for its own view of the plan
(wd_plan_decomposition: host logic only, the same code wd_assemble and the
V-cycle's exchanges use), the views are all-gathered through the torch
process group, and the invariants are checked here from first principles:

  * all ranks agree on the hierarchy and the gather level; levels before the
    gather level are distributed, the rest replicated;
  * on a distributed level the owned rows partition the level's rows in rank
    order (>= 4 each), every rank holds its owned rows plus 2 halo rows per
    side (clipped at the grid), and a coarse rank owns exactly the coarse rows
    whose kept fine row (horizontal kept set {0, 2, ...} U {n - 1}, reading
    C5) it owns on the fine level;
  * every send of a w-row exchange has a matching receive at the peer (same
    rows, same count), senders send owned rows, and each rank receives exactly
    the w rows next to its owned range on each side that has a neighbour;
  * on the gather level the ranks' compute slices partition the level's rows;
    after it every rank computes everything.
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

HALO = 2
MIN_OWNED = 4

# (name, dims, a, h1, h3, options)
GRIDS = [
    ("paper", (3001, 3001, 16), (1, 1, 10), 33.0, 10.0 * 1.25 ** np.arange(15), {}),
    ("medium", (1001, 1001, 16), (1, 1, 10), 30.0, 10.0 * 1.25 ** np.arange(15), {}),
    ("medium_nogather", (1001, 1001, 16), (1, 1, 10), 30.0, 10.0 * 1.25 ** np.arange(15),
     {"gather_below_nodes": 0}),
    ("odd_rows", (517, 403, 9), (1, 1, 1), 20.0, 5.0 * 1.2 ** np.arange(8),
     {"gather_below_nodes": 0, "coarsest_max_free": 300}),
    ("small", (129, 129, 11), (1, 1, 10), 50.0, 10.0 * 1.2 ** np.arange(10), {}),
]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2101_08453_b200 as wd
    res = {}
    for name, dims, a, h1, h3, kw in GRIDS:
        if dims[1] // world < MIN_OWNED:
            continue
        for w in (1, 2):
            plan = wd.wd_plan_decomposition(dims, a, h1, h3, world, rank, w=w,
                                            opt=wd.default_options(**kw))
            got = [None] * world
            dist.all_gather_object(got, plan)
            res[(name, w)] = got
    out[rank] = res
    dist.destroy_process_group()


def _kept(n):
    pos = list(range(0, n, 2))
    if pos[-1] != n - 1:
        pos.append(n - 1)
    return pos


def check_plans(plans, w):
    R = len(plans)
    p0 = plans[0]
    nl = p0["nlevels"]
    for p in plans:
        assert p["nlevels"] == nl and p["gather"] == p0["gather"]
        assert [lv["dims"] for lv in p["levels"]] == [lv["dims"] for lv in p0["levels"]]
    gather = p0["gather"] if p0["gather"] >= 0 else nl
    assert 1 <= gather
    recv_rows = {}
    for l in range(nl):
        n1, n2, n3 = p0["levels"][l]["dims"]
        dists = [p["levels"][l]["dist"] for p in plans]
        assert all(d == (l < gather) for d in dists), (l, gather, dists)
        if l < gather:
            own = [p["levels"][l]["owned"] for p in plans]
            assert own[0][0] == 0 and own[-1][1] == n2
            for r in range(R):
                a, b = own[r]
                assert b - a >= MIN_OWNED
                if r + 1 < R:
                    assert own[r + 1][0] == b
                assert plans[r]["levels"][l]["held"] == (max(a - HALO, 0), min(b + HALO, n2))
            if l > 0:   # coarse ownership follows the fine owner of the kept row
                fn2 = p0["levels"][l - 1]["dims"][1]
                pos = _kept(fn2) if n2 < fn2 else list(range(fn2))
                assert len(pos) == n2
                fown = [p["levels"][l - 1]["owned"] for p in plans]
                for r in range(R):
                    want = [J for J in range(n2) if fown[r][0] <= pos[J] < fown[r][1]]
                    assert (want[0], want[-1] + 1) == own[r], (l, r)
        else:
            comp = [p["levels"][l]["owned"] for p in plans]
            for p in plans:
                assert p["levels"][l]["held"] == (0, n2)
            if l == gather:
                assert comp[0][0] == 0 and comp[-1][1] == n2
                for r in range(R - 1):
                    assert comp[r][1] == comp[r + 1][0]
            else:
                assert all(c == (0, n2) for c in comp)
        # messages of this level
        for r in range(R):
            mine = [m for m in plans[r]["msgs"] if m["level"] == l]
            if l >= gather:
                assert not mine
                continue
            a, b = plans[r]["levels"][l]["owned"]
            want_recv = set()
            if r > 0:
                want_recv |= set(range(a - w, a))
            if r < R - 1:
                want_recv |= set(range(b, b + w))
            got_recv = set()
            for m in mine:
                assert m["rows"] == w and m["peer"] in (r - 1, r + 1)
                rows = set(range(m["row0"], m["row0"] + m["rows"]))
                if m["send"]:
                    assert rows <= set(range(a, b))
                    match = [q for q in plans[m["peer"]]["msgs"]
                             if q["level"] == l and q["peer"] == r and not q["send"]
                             and q["row0"] == m["row0"] and q["rows"] == m["rows"]]
                    assert len(match) == 1, (l, r, m)
                else:
                    got_recv |= rows
            assert got_recv == want_recv, (l, r)
            recv_rows[(l, r)] = got_recv
    nsend = sum(m["send"] for p in plans for m in p["msgs"])
    nrecv = sum(not m["send"] for p in plans for m in p["msgs"])
    assert nsend == nrecv


@pytest.mark.parametrize("world", [2, 3, 4, 8])
def test_decomposition_schedule_gloo(world):
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    res = out[0]
    assert res
    for (name, w), plans in res.items():
        assert len(plans) == world
        check_plans(plans, w)
        # every rank saw the same all-gathered views
        for r in range(1, world):
            assert out[r][(name, w)] == plans
    # the paper grid at 8 ranks distributes at least three levels
    if world == 8:
        assert res[("paper", 1)][0]["gather"] >= 3


@pytest.mark.parametrize("grid", [g[0] for g in GRIDS])
def test_plan_single_rank_matches_oracle_planner(grid):
    """One rank: no messages, held = owned = all rows, and the level dims are
    those of the oracle's planner (oracle.plan_level, readings
    C1-C5) iterated from the same (h1, h3) until <= coarsest_max_free free
    unknowns or nothing coarsens."""
    import oracle
    import paper_2101_08453_b200 as wd
    name, dims, a, h1, h3, kw = [g for g in GRIDS if g[0] == grid][0]
    opt = wd.default_options(**kw)
    p = wd.wd_plan_decomposition(dims, a, h1, h3, 1, 0, opt=opt)
    assert p["msgs"] == [] and p["gather"] == -1
    want = [tuple(dims)]
    hh1, hh3 = h1, np.asarray(h3, dtype=float)
    n1, n2, n3 = dims
    while (n1 - 2) * (n2 - 2) * (n3 - 1) > opt.coarsest_max_free:
        pl = oracle.plan_level(hh1, hh3, a, n1=n1, n2=n2)
        if not pl["coarsens"]:
            break
        if pl["horizontal"]:
            n1, n2 = len(_kept(n1)), len(_kept(n2))
        n3 = len(pl["kept"])
        hh1, hh3 = pl["h1"], pl["h3"]
        want.append((n1, n2, n3))
    assert [lv["dims"] for lv in p["levels"]] == want
    for lv in p["levels"]:
        assert lv["held"] == (0, lv["dims"][1]) and lv["owned"] == (0, lv["dims"][1])


def test_plan_rejects_thin_slabs():
    import paper_2101_08453_b200 as wd
    with pytest.raises(wd.WDError) as e:
        wd.wd_plan_decomposition((17, 17, 9), (1, 1, 1), 30.0, [5.0] * 8, 8, 0)
    assert e.value.code == wd.WD_E_INVAL
