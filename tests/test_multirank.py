"""World-size-2 row-slab path on CPU (gloo): slab cover, stitched CSR == full, checksum all-reduce."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1904_06971_b200.slabs import allreduce_checksum, csr_checksum, plane_slabs, stitch, weighted_plane_slabs


def test_plane_slabs_cover_rows_contiguously():
    ms = (11, 9, 13)
    for world in (1, 2, 4, 8):
        sl = plane_slabs(ms, world)
        assert sl[0][0] == 0 and sl[-1][1] == int(np.prod(ms))
        assert all(a[1] == b[0] for a, b in zip(sl, sl[1:]))
        assert all((hi - lo) % (11 * 9) == 0 for lo, hi in sl)
    with pytest.raises(ValueError):
        plane_slabs(ms, 14)


def test_weighted_slabs_balance_cost():
    cost = np.r_[np.full(6, 10.0), np.ones(20), np.full(6, 10.0)]
    sl = weighted_plane_slabs(cost, 100, 2)
    assert sl[0][0] == 0 and sl[-1][1] == 3200 and sl[0][1] == sl[1][0]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import torch.distributed as dist

    from oracle import surriga_oracle as O
    import paper_1904_06971_b200 as pkg

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    disc = pkg.make_discretization(pkg.twisted_cube_standin(), 2, (5, 4, 6))
    prob = O.problem_from_disc(pkg.FormKind.POISSON, disc)
    lo, hi = plane_slabs(prob.ms, world)[rank]
    ip, ix, d, _, _ = O.assemble(prob, rows=np.arange(lo, hi))
    sl_ip = ip[lo:hi + 1] - ip[lo]
    cs = allreduce_checksum(csr_checksum(sl_ip, d), dist)
    gathered = [None] * world
    dist.all_gather_object(gathered, (sl_ip, ix, d))
    if rank == 0:
        q.put((cs, gathered))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_slabs_gloo_equal_full():
    from oracle import surriga_oracle as O
    import paper_1904_06971_b200 as pkg

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    cs, parts = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    disc = pkg.make_discretization(pkg.twisted_cube_standin(), 2, (5, 4, 6))
    ip, ix, d, _, _ = O.assemble(O.problem_from_disc(pkg.FormKind.POISSON, disc))
    sip, six, sd = stitch(parts)
    assert np.array_equal(sip, ip) and np.array_equal(six, ix)
    assert np.array_equal(sd.view(np.int64), d.view(np.int64))  # restricted rows are bitwise the full rows
    full = csr_checksum(ip, d)
    assert cs[0] == full[0]
    assert np.allclose(cs[1:], full[1:], rtol=1e-12, atol=1e-12)


def test_surrogate_plane_cost_rows_and_balance():
    # the per-plane row classes of the cost model add up to the exact plan (surrogate_plan), and
    # cost-weighted slabs balance the surrogate of config 5 across 8 ranks better than equal planes
    import paper_1904_06971_b200 as pkg
    from paper_1904_06971_b200.configs import CONFIGS
    from paper_1904_06971_b200.slabs import SURROGATE_ROW_COST, surrogate_plane_cost
    from paper_1904_06971_b200.surrogate import build_sampling_lattice

    cfg = CONFIGS[5]
    disc = pkg.make_discretization(cfg.geom(), cfg.p, cfg.spans)
    ms = tuple(kv.m for kv in disc.space.kvs)
    lat = build_sampling_lattice(disc.space.kvs, cfg.M)
    per = int(np.prod(ms[:-1]))
    cq, ci, c0 = SURROGATE_ROW_COST["poisson"]
    cost = surrogate_plane_cost(ms, cfg.p, lat.indices, "poisson")
    interp = (cost - c0 * per - cq * per) / (ci - cq)  # invert cost = cq quad + ci interp + c0 per
    plan = pkg.surrogate_plan(disc, pkg.ConstantSampling(cfg.M), cfg.q)
    assert round(interp.sum()) == plan.interp_rows
    def imbalance(sl):
        c = [cost[lo // per:hi // per].sum() for lo, hi in sl]
        return max(c) / np.mean(c)
    assert imbalance(weighted_plane_slabs(cost, per, 8)) < 1.08 < 1.3 < imbalance(plane_slabs(ms, 8))
    assert imbalance(weighted_plane_slabs(cost, per, 4)) < 1.05


def test_halo_balanced_slabs_beat_per_plane_balancing_under_the_halo_cost():
    """Slabs that pay for their p-plane halo (the surrogate recomputes its quadrature rows): the dynamic
    program is never worse than per-plane balancing under that cost, covers every plane once and is
    exact on a case small enough to enumerate."""
    import itertools

    import paper_1904_06971_b200 as pkg
    from paper_1904_06971_b200.configs import CONFIGS
    from paper_1904_06971_b200.slabs import halo_balanced_plane_slabs, job_slabs, surrogate_plane_cost
    from paper_1904_06971_b200.surrogate import build_sampling_lattice

    def slab_cost(cost, halo, p, per, sl):
        out = []
        for lo, hi in sl:
            a, b = lo // per, hi // per
            out.append(cost[a:b].sum() + halo[max(a - p, 0):a].sum() + halo[b:b + p].sum())
        return max(out)

    cfg = CONFIGS[5]
    disc = pkg.make_discretization(cfg.geom(), cfg.p, cfg.spans)
    ms = tuple(kv.m for kv in disc.space.kvs)
    lat = build_sampling_lattice(disc.space.kvs, cfg.M)
    per = int(np.prod(ms[:-1]))
    for form in ("poisson", "mass"):
        cost, halo = surrogate_plane_cost(ms, cfg.p, lat.indices, form, parts=True)
        for world in (2, 4, 8):
            new = halo_balanced_plane_slabs(cost, halo, cfg.p, per, world)
            assert new[0][0] == 0 and new[-1][1] == per * ms[-1]
            assert all(new[r][1] == new[r + 1][0] and new[r][1] > new[r][0] for r in range(world - 1))
            old = weighted_plane_slabs(cost, per, world)
            assert slab_cost(cost, halo, cfg.p, per, new) <= slab_cost(cost, halo, cfg.p, per, old) * (1 + 1e-12)
            assert job_slabs(ms, cfg.p, world, "surrogate", form, lat.indices) == new
    # the all-quadrature boundary planes of config 5 make the halo matter at 8 slabs
    cost, halo = surrogate_plane_cost(ms, cfg.p, lat.indices, "poisson", parts=True)
    assert slab_cost(cost, halo, cfg.p, per, halo_balanced_plane_slabs(cost, halo, cfg.p, per, 8)) < \
        0.9 * slab_cost(cost, halo, cfg.p, per, weighted_plane_slabs(cost, per, 8))
    # exactness: brute force over every cut set of a small case
    rng = np.random.default_rng(5)
    c, h = rng.random(11) + 0.1, 3 * rng.random(11)
    best = min(slab_cost(c, h, 2, 1, [(a, b) for a, b in zip((0,) + cuts, cuts + (11,))])
               for cuts in itertools.combinations(range(1, 11), 3))
    assert abs(slab_cost(c, h, 2, 1, halo_balanced_plane_slabs(c, h, 2, 1, 4)) - best) < 1e-12
