"""Row slabs on the GPU library: the surrogate's strategy B (each slab assembles only
its own lattice rows; the sample table is completed by an exchange) and world-size-2 runs of the
library in two processes sharing one GPU over gloo (the CPU stand-in for the NCCL group of one
8-GPU box: the exchange and the checksum all-reduce are the only collectives; no kernel of one
rank waits on the other's).  Every stitched result must be bitwise the whole-matrix result."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

CASES = [("twisted", 3, (22, 21, 40), "poisson", 4), ("twisted", 3, (22, 21, 40), "mass", 4),
         ("twisted", 2, (18, 17, 33), "poisson", 3), ("annulus", 3, (40, 90), "poisson", 8)]


def _geom(name):
    import paper_1904_06971_b200 as pkg

    return pkg.twisted_cube_standin() if name == "twisted" else pkg.quarter_annulus(1.0, 2.0)


def _host(res):
    try:
        return res.to_host()
    finally:
        res.free()


@pytest.mark.gpu
@pytest.mark.parametrize("geom,p,spans,form,M", CASES)
@pytest.mark.parametrize("world", [2, 3])
def test_gpu_surrogate_strategy_b_in_process(geom, p, spans, form, M, world):
    """begin on every slab, exchange the owned lattice columns between the device tables (here by
    device copies in one process), finish: stitched == whole, bitwise; counts add up."""
    import torch

    import paper_1904_06971_b200 as pkg
    from paper_1904_06971_b200 import _lib
    from paper_1904_06971_b200.slabs import _device_view, job_slabs, lattice_owners, stitch
    from paper_1904_06971_b200.surrogate import DEFAULT_MODE, build_sampling_lattice, surrogate_device

    disc = pkg.make_discretization(_geom(geom), p, spans)
    fk = pkg.FormKind(form)
    mode = DEFAULT_MODE[form].value
    whole, wst, _ = surrogate_device(fk, disc, M, 3, mode)
    wip, wix, wd = _host(whole)
    ms = tuple(kv.m for kv in disc.space.kvs)
    lat = build_sampling_lattice(disc.space.kvs, M)
    slabs = job_slabs(ms, p, world, "surrogate", form, lat.indices)
    owner = lattice_owners(ms, lat.indices, slabs)
    # phase 1 on every slab; each table keeps only its own columns
    tables = []
    states = []
    for r, sl in enumerate(slabs):
        import ctypes as C

        pr, keep, _, _ = pkg.assembly.problem_arrays(fk, disc, 1.0)
        from paper_1904_06971_b200.surrogate import _fit_params, tilde_domain

        spp, keep2, _ = _fit_params(disc, lat, tilde_domain(p, ms), 3, mode, M)
        ex = pkg.assembly._exec(None, None, sl)
        state, table, nlat = C.c_void_p(), C.c_void_p(), C.c_int64()
        _lib.check(_lib.lib().sg_surrogate_begin(C.byref(pr), C.byref(spp), C.byref(ex), C.byref(state),
                                                 C.byref(table), C.byref(nlat)))
        P = (2 * p + 1) ** len(ms)
        t = _device_view(table.value, (P, nlat.value), torch.device("cuda", 0))
        own = np.flatnonzero(owner == r)
        other = np.flatnonzero(owner != r)
        assert torch.all(t[:, torch.as_tensor(other, device="cuda")] == 0)
        tables.append(t)
        states.append((state, spp, keep, keep2))
    full = torch.zeros_like(tables[0])
    for r, t in enumerate(tables):
        own = torch.as_tensor(np.flatnonzero(owner == r), device="cuda")
        full[:, own] = t[:, own]
    for t in tables:
        t.copy_(full)
    torch.cuda.synchronize()
    parts = []
    n_interp = 0
    for state, spp, keep, keep2 in states:
        import ctypes as C

        h, st = C.c_void_p(), _lib.SgSurrogateStats()
        _lib.check(_lib.lib().sg_surrogate_finish(state, C.byref(spp), C.byref(h), C.byref(st)))
        parts.append(_host(_lib.Result(h.value)))
        n_interp += st.n_interp_entries
    ip, ix, d = stitch(parts)
    assert np.array_equal(ip, wip) and np.array_equal(ix, wix)
    assert np.array_equal(d.view(np.int64), wd.view(np.int64))
    assert n_interp == wst.n_interp_entries


@pytest.mark.gpu
@pytest.mark.parametrize("geom,p,spans,form,M", CASES[:2])
def test_gpu_surrogate_slab_single_call_equals_whole(geom, p, spans, form, M):
    """A slab call without an exchange assembles the other slabs' lattice rows itself (row-restricted
    quadrature): stitched == whole, bitwise, and its work arrays cover only the slab and its halo."""
    import paper_1904_06971_b200 as pkg
    from paper_1904_06971_b200.slabs import job_slabs, stitch
    from paper_1904_06971_b200.surrogate import DEFAULT_MODE, build_sampling_lattice, surrogate_device

    disc = pkg.make_discretization(_geom(geom), p, spans)
    fk = pkg.FormKind(form)
    mode = DEFAULT_MODE[form].value
    wip, wix, wd = _host(surrogate_device(fk, disc, M, 3, mode)[0])
    ms = tuple(kv.m for kv in disc.space.kvs)
    lat = build_sampling_lattice(disc.space.kvs, M)
    parts = [_host(surrogate_device(fk, disc, M, 3, mode, slab=sl)[0])
             for sl in job_slabs(ms, p, 4, "surrogate", form, lat.indices)]
    ip, ix, d = stitch(parts)
    assert np.array_equal(ip, wip) and np.array_equal(ix, wix)
    assert np.array_equal(d.view(np.int64), wd.view(np.int64))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _rank_worker(rank, world, port, q):
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import torch
    import torch.distributed as dist

    import paper_1904_06971_b200 as pkg
    from paper_1904_06971_b200.slabs import allreduce_checksum, exchange_samples, job_slabs, lattice_owners
    from paper_1904_06971_b200.surrogate import DEFAULT_MODE, build_sampling_lattice, surrogate_device

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    disc = pkg.make_discretization(pkg.twisted_cube_standin(), 3, (22, 21, 40))
    ms = tuple(kv.m for kv in disc.space.kvs)
    lat = build_sampling_lattice(disc.space.kvs, 4)
    out = {}
    for form in ("poisson", "mass"):
        fk = pkg.FormKind(form)
        sl = job_slabs(ms, 3, world, "full", form)[rank]
        res, _, _ = pkg.assemble_device(fk, disc, slab=sl)
        cs_full = allreduce_checksum(res.checksum(), dist)
        out[(form, "full")] = (res.to_host(), cs_full)
        res.free()
        slabs = job_slabs(ms, 3, world, "surrogate", form, lat.indices)
        ex = exchange_samples(lattice_owners(ms, lat.indices, slabs), dist)
        res, st, _ = surrogate_device(fk, disc, 4, 3, DEFAULT_MODE[form].value, slab=slabs[rank], lattice=lat,
                                      exchange=ex)
        cs = allreduce_checksum(res.checksum(), dist)
        out[(form, "surrogate")] = (res.to_host(), cs)
        res.free()
    gathered = [None] * world
    dist.all_gather_object(gathered, out)
    if rank == 0:
        q.put(gathered)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
def test_gpu_two_ranks_share_one_gpu_gloo():
    import paper_1904_06971_b200 as pkg
    from paper_1904_06971_b200.slabs import stitch
    from paper_1904_06971_b200.surrogate import DEFAULT_MODE, surrogate_device

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    gathered = q.get(timeout=600)
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    disc = pkg.make_discretization(pkg.twisted_cube_standin(), 3, (22, 21, 40))
    for form in ("poisson", "mass"):
        fk = pkg.FormKind(form)
        for path in ("full", "surrogate"):
            if path == "full":
                res = pkg.assemble_device(fk, disc)[0]
            else:
                res = surrogate_device(fk, disc, 4, 3, DEFAULT_MODE[form].value)[0]
            cs_whole = res.checksum()
            wip, wix, wd = _host(res)
            ip, ix, d = stitch([g[(form, path)][0] for g in gathered])
            assert np.array_equal(ip, wip) and np.array_equal(ix, wix), (form, path)
            assert np.array_equal(d.view(np.int64), wd.view(np.int64)), (form, path)
            cs = gathered[0][(form, path)][1]
            assert cs[0] == cs_whole[0]
            assert np.allclose(cs[1:], cs_whole[1:], rtol=1e-12, atol=1e-300)
