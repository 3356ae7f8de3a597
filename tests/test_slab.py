"""Zero-communication z-slab partition (paper_1801_08914_b200/slab.py).

CPU: the partition's host logic against the oracle's port of the reference
(oracle/hdr_oracle.c, port_hybridize): every rank hybridizes its ghosted sub-mesh,
its owned rows must tile the global rows exactly once, map to the same columns,
and carry bit-identical H / g values (each entry is the sum of at most two cell
contributions).  Plus the same assembled over a world-2 gloo group.
GPU: the product path per rank (one GPU, ranks run one after the other, no
waiting between them) against the single-mesh product and the double-double oracle."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1801_08914_b200 import slab
from oracle_lib import Oracle, rel_err

LOGU = "logu:1e-2:1e2"
CASES = [((3, 2, 6), 0, LOGU, 2), ((3, 2, 7), 0, LOGU, 3), ((2, 2, 4), 1, LOGU, 2), ((2, 3, 5), 1, LOGU, 4),
         ((2, 2, 3), 2, "logu:1e-3:1e3", 3)]


def _global(cells, k, coef, seed=7):
    o = Oracle(3, cells, k)
    o.gen_inputs(coef, seed)
    o.run("port_hybridize")
    return o


def _rank_part(plan, g_or):
    """The rank's share through the oracle (the stand-in for its GPU)."""
    o = Oracle(3, plan.sub_cells, plan.order)
    o.set_h(plan.sizes)
    n = g_or.size("n")
    a, b, f = plan.inputs(g_or.get("alpha"), g_or.get("beta"), g_or.get("f_hat"), n)
    o.set("alpha", a)
    o.set("beta", b)
    o.set("f_hat", f)
    o.run("port_hybridize")
    return o, plan.extract(o.getq("H.row_offsets"), o.get("H.values"), o.get("g"))


def test_slab_layers_split():
    for nz in (1, 5, 8, 13):
        for world in (1, 2, 3, 8):
            spans = [slab.slab_layers(nz, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == nz
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
            assert max(b - a for a, b in spans) - min(b - a for a, b in spans) <= 1


@pytest.mark.parametrize("cells,k,coef,world", CASES)
def test_slab_parts_tile_global_bit_exact(cells, k, coef, world):
    g_or = _global(cells, k, coef)
    m, _, ro_g, ci_g, hv_g = g_or.csr("H")
    gv_g = g_or.get("g")
    seen = np.zeros(m, np.int64)
    h_out, g_out = np.full(hv_g.size, np.nan), np.full(m, np.nan)
    for rank in range(world):
        plan = slab.SlabPlan(cells, k, world, rank)
        o, part = _rank_part(plan, g_or)
        _, _, ro_l, ci_l, _ = o.csr("H")
        for ls, gs, n in plan.row_ranges:
            seen[gs:gs + n] += 1
            # same rows, same columns (mapped), same order
            assert np.array_equal(plan.local_to_global_rows(np.arange(ls, ls + n)), np.arange(gs, gs + n))
            assert np.array_equal(np.diff(ro_l[ls:ls + n + 1]), np.diff(ro_g[gs:gs + n + 1]))
            assert np.array_equal(plan.local_to_global_rows(ci_l[ro_l[ls]:ro_l[ls + n]]),
                                  ci_g[ro_g[gs]:ro_g[gs + n]])
        slab.place(part, ro_g, h_out, g_out)
    assert np.all(seen == 1)  # every global row owned exactly once
    assert np.array_equal(h_out, hv_g) and np.array_equal(g_out, gv_g)


def test_slab_ghost_overhead():
    plan = slab.SlabPlan((64, 64, 64), 0, 8, 3)
    assert plan.sub_cells == (64, 64, 11) and (plan.z0, plan.z1) == (24, 32)
    edge = slab.SlabPlan((64, 64, 64), 0, 8, 0)
    assert edge.sub_cells == (64, 64, 10) and edge.g0 == 0


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cells, k = (3, 2, 5), 1
    g_or = _global(cells, k, LOGU)
    _, part = _rank_part(slab.SlabPlan(cells, k, world, rank), g_or)
    parts = [None] * world
    dist.all_gather_object(parts, part)  # assembly only; the hybridization needed no exchange
    if rank == 0:
        m, _, ro_g, _, hv_g = g_or.csr("H")
        h_out, g_out = np.zeros(hv_g.size), np.zeros(m)
        for p in parts:
            slab.place(p, ro_g, h_out, g_out)
        out["ok"] = bool(np.array_equal(h_out, hv_g) and np.array_equal(g_out, g_or.get("g")))
    dist.destroy_process_group()


@pytest.mark.timeout(180)
def test_slab_two_rank_gloo():
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
        assert out["ok"]


@pytest.mark.gpu
@pytest.mark.parametrize("cells,k,coef,world", [((8, 8, 8), 0, LOGU, 3), ((4, 4, 6), 1, LOGU, 2),
                                                ((3, 3, 4), 3, "checker:1e-2:1e2", 2)])
def test_slab_gpu_matches_single_mesh(cells, k, coef, world):
    from paper_1801_08914_b200 import Space
    o = Oracle(3, cells, k)
    o.gen_inputs(coef, 11)
    o.run("port_hybridize")
    o.run("dd_hybridize")
    a, b, f = o.get("alpha"), o.get("beta"), o.get("f_hat")
    sp = Space(3, cells, k)
    hv, gv = sp.hybridize(a, b, f).values()
    ro, _ = sp.pattern("H")
    h_out, g_out = np.full(hv.size, np.nan), np.full(gv.size, np.nan)
    for rank in range(world):
        slab.place(slab.hybridize_slab(slab.SlabPlan(cells, k, world, rank), a, b, f), ro, h_out, g_out)
    assert not np.isnan(h_out).any() and not np.isnan(g_out).any()
    assert rel_err(h_out, hv) <= 1e-13 and rel_err(g_out, gv) <= 1e-13
    assert rel_err(h_out, o.get("H.values_dd")) <= 1e-11 and rel_err(g_out, o.get("g_dd")) <= 1e-11
