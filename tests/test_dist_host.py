"""Host logic of the row-strip decomposition on the CPU: the plan computed by
libhelm (helm_dist_plan, host-only) and, over a real world_size-2 `gloo` process group, the
exchange pattern of the NCCL transport (GHOST owned rows to each neighbour, rank-summed dots,
all-gather of the replicated level) applied to the oracle's operators on each rank's block.
No GPU: the CUDA kernels are exercised by tests/test_gpu_dist.py."""
import os
import socket

import numpy as np
import pytest

GHOST = 6   # dist.cuh


def _lib():
    from paper_2308_06152_b200 import helm
    return helm


def _window(s, e, dirichlet):
    H = e - s
    ws = s // 2
    return ws, ws + ((H - 1) // 2 if dirichlet else (H + 1) // 2)


PLANS = [(n, bc, P, mr) for n, bc in ((63, "dirichlet"), (127, "dirichlet"), (639, "dirichlet"), (65, "sommerfeld"),
                                       (257, "sommerfeld"), (1023, "dirichlet"))
         for P in (1, 2, 3, 4, 5, 8) for mr in (6, 16)]


@pytest.mark.parametrize("n,bc,P,mr", PLANS)
def test_plan_invariants(n, bc, P, mr):
    helm = _lib()
    try:
        D, rows = helm.dist_plan(n, n, 1.0 / (n + 1), bc, P, {"dist_min_rows": mr})
    except helm.HelmError as e:
        assert "too small" in str(e)
        return
    d = bc == "dirichlet"
    o = 1 if d else 0
    ny = [rl[-1][1] for rl in rows]   # the last rank owns up to the end
    assert 1 <= D <= len(rows) - 2
    for l, rl in enumerate(rows):
        # owned rows tile the level, in rank order
        assert rl[0][0] == 0 and rl[-1][1] == ny[l]
        assert all(rl[q][1] == rl[q + 1][0] for q in range(P - 1))
        if l > 0:   # coarse row J belongs to the owner of its coincident fine row 2J + o
            for q in range(P):
                for J in (rl[q][0], rl[q][1] - 1):
                    if rl[q][0] <= J < rl[q][1]:
                        f = rows[l - 1][q]
                        assert f[0] <= 2 * J + o < f[1] or (2 * J + o >= ny[l - 1] and q == P - 1)
    for l in range(D + 1):
        for q, (a, b, s, e) in enumerate(rows[l]):
            assert b - a >= max(GHOST, mr)
            assert s % 2 == 0 and (e - s) % 2 == 1 and 0 <= s and e <= ny[l]
            assert s <= max(0, a - GHOST) and e >= min(ny[l], b + GHOST)
            ws, we = _window(s, e, d)
            c = rows[l + 1][q]
            if l < D:   # the coarse block contains the window of the fine block
                assert c[2] <= ws and we <= c[3]
            else:       # level D+1 entry is that window
                assert (c[2], c[3]) == (ws, we) and we <= ny[l + 1]
            # the window holds the coarse owned rows and 2 rows around them (transfer radius)
            assert ws <= max(0, c[0] - 2) and we >= min(ny[l + 1], c[1] + 2)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank_main(rank, world, port, q):
    import torch
    import torch.distributed as dist
    import oracle
    from workloads import random_field, random_k
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        helm = _lib()
        res = {}
        for n, bc in ((63, "dirichlet"), (65, "sommerfeld")):
            h = 1.0 / (n + 1)
            k = random_k((n, n), 5, 5, 40)
            u = random_field((n, n), 6)
            D, rows = helm.dist_plan(n, n, h, bc, world, {"dist_min_rows": 6})
            a, b, s, e = rows[0][rank]
            blk = np.zeros((e - s, n), complex)
            blk[a - s:b - s] = u[a:b]            # only the owned rows are known locally
            # halo exchange, NCCL transport pattern: GHOST owned rows to each neighbour
            reqs = []
            up = torch.from_numpy(blk[a - s:a - s + GHOST].view(np.float64).copy())
            dn = torch.from_numpy(blk[b - s - GHOST:b - s].view(np.float64).copy())
            rup = torch.empty_like(up)
            rdn = torch.empty_like(dn)
            if rank > 0:
                reqs += [dist.isend(up, rank - 1), dist.irecv(rup, rank - 1)]
            if rank < world - 1:
                reqs += [dist.isend(dn, rank + 1), dist.irecv(rdn, rank + 1)]
            for r in reqs:
                r.wait()
            if rank > 0:
                blk[a - s - GHOST:a - s] = rup.numpy().view(complex)
            if rank < world - 1:
                blk[b - s:b - s + GHOST] = rdn.numpy().view(complex)
            # the oracle's A on the block as a grid of its own (its edge rows get boundary
            # treatment): the owned rows must equal the global operator's, since the block
            # edges are >= GHOST rows away from them
            y_blk = oracle.apply_A(blk, k[s:e], h, bc)
            y_glob = oracle.apply_A(u, k, h, bc)
            err = np.abs(y_blk[a - s:b - s] - y_glob[a:b]).max() / np.abs(y_glob).max()
            # rank-summed dot (allreduce) equals the global dot
            part = torch.tensor([np.vdot(u[a:b], y_glob[a:b]).real, np.vdot(u[a:b], y_glob[a:b]).imag])
            dist.all_reduce(part)
            gdot = np.vdot(u, y_glob)
            derr = abs(complex(part[0].item(), part[1].item()) - gdot) / abs(gdot)
            # all-gather of the replicated level D+1: every rank ends with the whole level
            cl = rows[D + 1]
            mine = torch.from_numpy(np.ascontiguousarray(u[cl[rank][0]:cl[rank][1]]).view(np.float64).ravel())
            sizes = [2 * (cl[r][1] - cl[r][0]) * n for r in range(world)]
            bufs = []
            for r in range(world):   # one broadcast per owner, as the NCCL transport
                t_ = mine.clone() if r == rank else torch.empty(sizes[r], dtype=torch.float64)
                dist.broadcast(t_, src=r)
                bufs.append(t_)
            full = np.concatenate([bb.numpy().view(complex).reshape(-1, n) for bb in bufs])
            gerr = np.abs(full - u[:full.shape[0]]).max()
            res[bc] = (float(err), float(derr), float(gerr), full.shape[0] == cl[-1][1])
        q.put((rank, res))
        dist.destroy_process_group()
    except BaseException as ex:   # noqa: BLE001
        q.put((rank, repr(ex)))


def test_gloo_world2_exchange_pattern():
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(60)
    for r in range(2):
        assert isinstance(out[r], dict), out[r]
        for bc, (err, derr, gerr, whole) in out[r].items():
            assert err < 1e-15, (r, bc, err)
            assert derr < 1e-13, (r, bc, derr)
            assert gerr == 0.0 and whole, (r, bc)


def _layout_rank(rank, world, port, q):
    import torch.distributed as dist
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        helm = _lib()
        res = {}
        for n, ny, bc, P in ((639, 1279, "dirichlet", 2), (2047, 8191, "dirichlet", 4), (257, 513, "sommerfeld", 3)):
            lay = helm.peer_layout(n, ny, 1.0 / (n + 1), bc, P, {"dist_levels": 3})
            allv = [None] * world
            dist.all_gather_object(allv, lay)
            # the IPC handle exchange of the peer transport: 64 opaque bytes per rank, rank order
            h = bytes([rank]) * 64
            hs = [None] * world
            dist.all_gather_object(hs, h)
            res[(n, ny, bc, P)] = (all(a == allv[0] for a in allv), lay,
                                   [x == bytes([r]) * 64 for r, x in enumerate(hs)])
        q.put((rank, res))
        dist.destroy_process_group()
    except BaseException as ex:   # noqa: BLE001
        q.put((rank, repr(ex)))


def test_gloo_world2_peer_layout_agrees():
    """The peer transport addresses a peer's slots by offsets it computes itself: every rank
    must derive the same arena layout from the global plan; the 64-byte IPC handles travel in
    rank order.  Slots are disjoint, 256-byte aligned and inside the arena."""
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_layout_rank, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(60)
    for r in range(2):
        assert isinstance(out[r], dict), out[r]
        for key, (same, lay, handles_ok) in out[r].items():
            assert same, key
            assert all(handles_ok), key
            total, offsets = lay[0], sorted(lay[1:4] + lay[5:])
            assert all(o % 256 == 0 and o < total for o in offsets), key
            assert len(set(offsets)) == len(offsets), key
