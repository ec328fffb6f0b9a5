"""Multi-GPU path on the CPU (world_size 2, gloo): the host-side plan of lpfem_halo_plan (the lists the library
uploads for its NCCL grouped send/recv after every write-back) is exchanged with torch.distributed
exactly as the device path does with NCCL, and every node of each rank's extended boxes must end up with the
owner's value; the gather of owned values reproduces the full field on rank 0.  The placement of subdomain
positions on ranks (lpfem_placement, LPT on box cells) is checked for balance against SURVEY 8(e)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

CASES = [
    # dim, fine cells per axis (region), subdomain grid, overlap cells
    (2, (64, 64), (4, 4), 8),    # cfg1 regions
    (2, (16, 16), (2, 2), 4),    # cfg0 regions
    (3, (16, 16, 16), (2, 2, 2), 4),  # cfg3 regions
    (3, (12, 12, 12), (3, 2, 2), 2),
]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _boxes(dim, n, m, ov, rank, world):
    import paper_2311_05170_b200 as P
    npos = int(np.prod(m))
    place = P.placement(dim, n, n, m, ov, world)
    out = []
    for s in range(npos):
        if place[s] != rank:
            continue
        rem, lo, hi = s, [], []
        for a in range(dim):
            pos = rem % m[a]
            rem //= m[a]
            core = n[a] // m[a]
            lo.append(2 * max(0, pos * core - ov))
            hi.append(2 * min(n[a], (pos + 1) * core + ov))
        out.append((lo, hi))
    return out


def _worker(rank, world, port, results):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist
    import paper_2311_05170_b200 as P
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ok = True
    msgs = []
    for dim, n, m, ov in CASES:
        for vertex in (False, True):
            shape = [(2 * k + 1) if not vertex else (k + 1) for k in n]
            N = int(np.prod(shape))
            truth = np.arange(N, dtype=np.float64) * 1.5 + 7.0
            field = np.full(N, np.nan)
            mine = P.halo_plan(dim, n, m, ov, rank, world, "owned", rank, vertex)
            field[mine] = truth[mine]
            reqs, bufs = [], []
            for peer in range(world):
                if peer == rank:
                    continue
                give = P.halo_plan(dim, n, m, ov, rank, world, "give", peer, vertex)
                need = P.halo_plan(dim, n, m, ov, rank, world, "need", peer, vertex)
                # lists must match the peer's view (computed independently on each rank)
                theirs = P.halo_plan(dim, n, m, ov, peer, world, "need", rank, vertex)
                if not np.array_equal(give, theirs):
                    ok = False
                    msgs.append(f"list mismatch {dim} {n} {peer}")
                sb = torch.from_numpy(field[give].copy())
                rb = torch.empty(len(need), dtype=torch.float64)
                reqs.append(dist.isend(sb, peer))
                reqs.append(dist.irecv(rb, peer))
                bufs.append((need, rb))
            for r in reqs:
                r.wait()
            for need, rb in bufs:
                field[need] = rb.numpy()
            # every node of my boxes now holds the owner's value
            for lo, hi in _boxes(dim, n, m, ov, rank, world):
                st = 2 if vertex else 1
                axes = [np.arange(lo[a], hi[a] + 1, st) // (2 if vertex else 1) for a in range(dim)]
                grid = np.meshgrid(*axes[::-1], indexing="ij")
                idx = np.zeros(grid[0].shape, dtype=np.int64)
                stride = 1
                for a in range(dim):
                    idx += grid[dim - 1 - a] * stride
                    stride *= shape[a]
                if not np.array_equal(field[idx.ravel()], truth[idx.ravel()]):
                    ok = False
                    msgs.append(f"halo values wrong {dim} {n} vertex={vertex}")
            # gather of owned values on rank 0 reproduces the field
            if rank == 0:
                full = field.copy()
                for peer in range(1, world):
                    own = P.halo_plan(dim, n, m, ov, rank, world, "owned", peer, vertex)
                    rb = torch.empty(len(own), dtype=torch.float64)
                    dist.recv(rb, peer)
                    full[own] = rb.numpy()
                if not np.array_equal(full, truth):
                    ok = False
                    msgs.append(f"gather wrong {dim} {n}")
            else:
                dist.send(torch.from_numpy(field[mine].copy()), 0)
    results[rank] = (ok, msgs)
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_halo_plan_exchange_gloo(world):
    from paper_2311_05170_b200 import build
    build.build()
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), results), nprocs=world, join=True)
    for r in range(world):
        ok, msgs = results[r]
        assert ok, msgs


def test_plan_partitions_nodes():
    """owned lists of all ranks partition the node set; halos only contain nodes owned by the peer."""
    from paper_2311_05170_b200 import build, halo_plan
    build.build()
    dim, n, m, ov, world = 2, (64, 64), (4, 4), 8, 4
    N = (2 * n[0] + 1) * (2 * n[1] + 1)
    allown = np.concatenate([halo_plan(dim, n, m, ov, 0, world, "owned", p) for p in range(world)])
    assert np.array_equal(np.sort(allown), np.arange(N))
    for r in range(world):
        for p in range(world):
            if p == r:
                continue
            need = halo_plan(dim, n, m, ov, r, world, "need", p)
            assert np.isin(need, halo_plan(dim, n, m, ov, r, world, "owned", p)).all()


def _box_cells(n, m, ov):
    """cells of every position's extended box (overlap clipped, C7), lexicographic positions"""
    dim = len(n)
    out = []
    for s in range(int(np.prod(m))):
        rem, c = s, 1
        for a in range(dim):
            pos = rem % m[a]
            rem //= m[a]
            core = n[a] // m[a]
            c *= min(n[a], (pos + 1) * core + ov) - max(0, pos * core - ov)
        out.append(c)
    return np.array(out)


@pytest.mark.parametrize("world", [2, 4, 8])
def test_placement_balance_cfg4_and_cfg2(world):
    """cfg4 (4x4x4 positions, boxes 18^3 .. 24^3) splits with every rank holding the same cell count
    (the octant balance: equal shape mix); cfg2 (8x8, boxes 48^2 .. 64^2) within 1% of the mean (contiguous
    blocks: 7% above it).  Every position placed exactly once, deterministically."""
    from paper_2311_05170_b200 import build, placement
    build.build()
    for dim, n, m, ov, tol in ((3, (48, 48, 48), (4, 4, 4), 6, 0.0), (2, (256, 256), (8, 8), 16, 0.01)):
        r = placement(dim, n, n, m, ov, world)
        assert r.min() == 0 and r.max() == world - 1
        w = 2 * _box_cells(n, m, ov)  # porous + conduit boxes
        load = np.array([w[r == k].sum() for k in range(world)])
        assert load.sum() == w.sum()
        assert load.max() <= (1 + tol) * load.mean(), (dim, world, load)
        assert np.array_equal(r, placement(dim, n, n, m, ov, world))
