"""Multi-rank host logic on CPU (gloo, world_size 2): the row-sharded SART of
SURVEY §8e — nnz-balanced row blocks from the product's partition_rows, a
per-iteration all-reduce of [A_g^T w_g | ||r_g||^2], identical updates on every
rank — must reproduce the unsharded oracle sart_solve. The GPU version of the
same decomposition is ss_plan_create_sharded (NCCL inside the library).

The peer-exchange protocol of ss_plan_create_sharded_x(SS_XCHG_PEER) is
modelled the same way: every rank's partial lands in the owner's receive row
(exchange_owned_columns), the owner sums the rows in rank order, updates its
range and pushes it to every replica; ||r||^2 is summed in rank order too, so
every rank's iterate is bitwise identical and equals the oracle."""
import os
import socket

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def csr_matvec(ptr, idx, val, x):
    rows = np.repeat(np.arange(len(ptr) - 1), np.diff(ptr))
    return np.bincount(rows, weights=val * x[idx], minlength=len(ptr) - 1)


def csr_rmatvec(ptr, idx, val, y, ncols):
    rows = np.repeat(np.arange(len(ptr) - 1), np.diff(ptr))
    return np.bincount(idx, weights=val * y[rows], minlength=ncols)


def sharded_sart(rank, world, ptr, idx, val, p, iters, relax, tol):
    import torch
    import torch.distributed as dist

    import paper_1902_10559_b200 as P
    rows, ncols = len(ptr) - 1, int(idx.max()) + 1
    bounds = P.symsplit.partition_rows(ptr, world)
    rb, re = int(bounds[rank]), int(bounds[rank + 1])
    lptr = ptr[rb:re + 1] - ptr[rb]
    lidx, lval = idx[ptr[rb]:ptr[re]], val[ptr[rb]:ptr[re]]
    # normalisers: local rows, global columns (every rank holds the same col sums)
    rsum = np.add.reduceat(np.abs(val), ptr[:-1]) if len(val) else np.zeros(rows)
    rsum[np.diff(ptr) == 0] = 0.0
    csum = np.bincount(idx, weights=np.abs(val), minlength=ncols)
    rinv = np.where(rsum > 0, 1.0 / np.where(rsum > 0, rsum, 1.0), 0.0)[rb:re]
    cinv = np.where(csum > 0, 1.0 / np.where(csum > 0, csum, 1.0), 0.0)
    pl = p[rb:re]
    pn2 = torch.tensor([float(pl @ pl)], dtype=torch.float64)
    dist.all_reduce(pn2)
    pnorm = float(np.sqrt(pn2.item()))
    x = np.zeros(ncols)
    hist = []
    for it in range(iters):
        r = pl - csr_matvec(lptr, lidx, lval, x)
        w = rinv * r
        buf = np.concatenate([csr_rmatvec(lptr, lidx, lval, w, ncols), [float(r @ r)]])
        t = torch.from_numpy(buf)
        dist.all_reduce(t)
        bp, r2 = t.numpy()[:-1], float(t.numpy()[-1])
        res = np.sqrt(r2)
        hist.append(res)
        if res <= tol * pnorm:
            break
        x = x + relax * (bp * cinv)
    return x, hist, (rb, re)


def peer_sharded_sart(rank, world, ptr, idx, val, p, iters, relax, tol):
    """The SS_XCHG_PEER data movement over gloo: all_gather stands in for the
    NVLink stores into the owners' receive rows and for the x pushes."""
    import torch
    import torch.distributed as dist

    import paper_1902_10559_b200 as P
    rows, ncols = len(ptr) - 1, int(idx.max()) + 1
    bounds = P.symsplit.partition_rows(ptr, world)
    rb, re = int(bounds[rank]), int(bounds[rank + 1])
    own = [P.symsplit.exchange_owned_columns(ncols, world, g) for g in range(world)]
    j0, j1 = own[rank]
    lptr = ptr[rb:re + 1] - ptr[rb]
    lidx, lval = idx[ptr[rb]:ptr[re]], val[ptr[rb]:ptr[re]]
    rsum = np.add.reduceat(np.abs(val), ptr[:-1]) if len(val) else np.zeros(rows)
    rsum[np.diff(ptr) == 0] = 0.0
    csum = np.bincount(idx, weights=np.abs(val), minlength=ncols)
    rinv = np.where(rsum > 0, 1.0 / np.where(rsum > 0, rsum, 1.0), 0.0)[rb:re]
    cinv = np.where(csum > 0, 1.0 / np.where(csum > 0, csum, 1.0), 0.0)
    pl = p[rb:re]
    pn2 = [torch.zeros(1, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(pn2, torch.tensor([float(pl @ pl)], dtype=torch.float64))
    pnorm = float(np.sqrt(sum(float(t.item()) for t in pn2)))  # run_group's rank order
    x = np.zeros(ncols)
    hist = []
    for it in range(iters):
        r = pl - csr_matvec(lptr, lidx, lval, x)
        w = rinv * r
        part = torch.from_numpy(csr_rmatvec(lptr, lidx, lval, w, ncols))
        recv = [torch.zeros(ncols, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(recv, part)          # receive row g <- rank g's partial
        r2s = [torch.zeros(1, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(r2s, torch.tensor([float(r @ r)], dtype=torch.float64))
        r2 = 0.0
        for t in r2s:                        # xr2_sum: rank order
            r2 += float(t.item())
        res = np.sqrt(r2)
        hist.append(res)
        if res <= tol * pnorm:
            break
        s_ = recv[0].numpy()[j0:j1].copy()   # rank-order sum of the owned range
        for g in range(1, world):
            s_ = s_ + recv[g].numpy()[j0:j1]
        mine = x[j0:j1] + relax * (s_ * cinv[j0:j1])
        width = max(e - b for b, e in own)
        pushed = [torch.zeros(width, dtype=torch.float64) for _ in range(world)]
        buf = torch.zeros(width, dtype=torch.float64)
        buf[:j1 - j0] = torch.from_numpy(mine)
        dist.all_gather(pushed, buf)         # every owner's range into every replica
        x = np.concatenate([pushed[g].numpy()[:own[g][1] - own[g][0]] for g in range(world)])
    return x, hist, own


def peer_pair_sharded_sart(rank, world, m1, m2, p1, p2, iters, relax, tol):
    """The row-sharded PAIR (ss_plan_create_sharded_pair): both folded systems
    split into the same row blocks (partition_rows of the shared pattern), one
    {u1, u2} receive row per rank and owner, ||r_g||^2 pairs summed in rank
    order, each system with its own check-before-update stop."""
    import torch
    import torch.distributed as dist

    import paper_1902_10559_b200 as P
    mats = [m1, m2]
    ps = [p1, p2]
    ptr0 = mats[0][0]
    rows, ncols = len(ptr0) - 1, int(max(m[1].max() for m in mats)) + 1
    bounds = P.symsplit.partition_rows(ptr0, world)
    rb, re = int(bounds[rank]), int(bounds[rank + 1])
    own = [P.symsplit.exchange_owned_columns(ncols, world, g) for g in range(world)]
    j0, j1 = own[rank]
    loc, rinv, cinv, pl, pnorm = [], [], [], [], []
    for (ptr, idx, val), p in zip(mats, ps):
        loc.append((ptr[rb:re + 1] - ptr[rb], idx[ptr[rb]:ptr[re]], val[ptr[rb]:ptr[re]]))
        rsum = np.add.reduceat(np.abs(val), ptr[:-1])
        rsum[np.diff(ptr) == 0] = 0.0
        csum = np.bincount(idx, weights=np.abs(val), minlength=ncols)
        rinv.append(np.where(rsum > 0, 1.0 / np.where(rsum > 0, rsum, 1.0), 0.0)[rb:re])
        cinv.append(np.where(csum > 0, 1.0 / np.where(csum > 0, csum, 1.0), 0.0))
        pl.append(p[rb:re])
        g2 = [torch.zeros(1, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(g2, torch.tensor([float(p[rb:re] @ p[rb:re])], dtype=torch.float64))
        pnorm.append(float(np.sqrt(sum(float(t.item()) for t in g2))))
    x = [np.zeros(ncols), np.zeros(ncols)]
    hist = [[], []]
    on = [True, True]
    for it in range(iters):
        if not any(on):
            break
        part = np.zeros((ncols, 2))
        r2 = np.zeros(2)
        for q in range(2):
            if not on[q]:
                continue
            lp, li, lv = loc[q]
            r = pl[q] - csr_matvec(lp, li, lv, x[q])
            part[:, q] = csr_rmatvec(lp, li, lv, rinv[q] * r, ncols)
            r2[q] = float(r @ r)
        recv = [torch.zeros(ncols * 2, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(recv, torch.from_numpy(part.reshape(-1)))  # {u1, u2} rows
        r2s = [torch.zeros(2, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(r2s, torch.from_numpy(r2))
        width = max(e - b for b, e in own)
        for q in range(2):
            if not on[q]:
                continue
            t = 0.0
            for g in range(world):                        # rank order
                t += float(r2s[g][q].item())
            res = np.sqrt(t)
            hist[q].append(res)
            if res <= tol * pnorm[q]:
                on[q] = False                             # this system stops here
                continue
            s_ = recv[0].numpy().reshape(ncols, 2)[j0:j1, q].copy()
            for g in range(1, world):
                s_ = s_ + recv[g].numpy().reshape(ncols, 2)[j0:j1, q]
            mine = x[q][j0:j1] + relax * (s_ * cinv[q][j0:j1])
            buf = torch.zeros(width, dtype=torch.float64)
            buf[:j1 - j0] = torch.from_numpy(mine)
            pushed = [torch.zeros(width, dtype=torch.float64) for _ in range(world)]
            dist.all_gather(pushed, buf)
            x[q] = np.concatenate([pushed[g].numpy()[:own[g][1] - own[g][0]]
                                   for g in range(world)])
    return x, hist, (rb, re)


def peer_pair_worker(rank, world, port, q, iters, tol):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch.distributed as dist

    import pyoracle as O
    from helpers import oracle_workload
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        w, cfg, a, csr, f_true, p = oracle_workload(1, literal=True)
        f1, f2 = O.fold_rows_csr(csr)
        p1, p2 = O.split_rhs(p)
        q.put((rank, peer_pair_sharded_sart(rank, world, f1.arrays(), f2.arrays(), p1, p2,
                                            iters, w.relaxation, tol)))
    finally:
        dist.destroy_process_group()


def peer_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch.distributed as dist

    import pyoracle as O
    from helpers import oracle_workload
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        w, cfg, a, csr, f_true, p = oracle_workload(1, literal=True)
        f1, f2 = O.fold_rows_csr(csr)
        p1, p2 = O.split_rhs(p)
        out = {}
        for name, m, pp in (("A1", f1, p1), ("A2", f2, p2)):
            ptr, idx, val = m.arrays()
            out[name] = peer_sharded_sart(rank, world, ptr, idx, val, pp, 30, w.relaxation, 0.0)
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch.distributed as dist

    import pyoracle as O
    from helpers import oracle_workload
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        w, cfg, a, csr, f_true, p = oracle_workload(1, literal=True)
        f1, f2 = O.fold_rows_csr(csr)
        p1, p2 = O.split_rhs(p)
        out = {}
        for name, m, pp in (("A1", f1, p1), ("A2", f2, p2)):
            ptr, idx, val = m.arrays()
            x, hist, rng = sharded_sart(rank, world, ptr, idx, val, pp, 30, w.relaxation, 0.0)
            out[name] = (x, hist, rng)
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_row_sharded_sart_matches_unsharded_oracle():
    import torch.multiprocessing as mp

    import pyoracle as O
    from helpers import oracle_workload
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    results = dict(q.get(timeout=300) for _ in range(world))
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    w, cfg, a, csr, f_true, p = oracle_workload(1, literal=True)
    split = O.split_system(a, p, 0.0)
    for name, m, pp in (("A1", split.a1, split.p1), ("A2", split.a2, split.p2)):
        want = O.sart_solve(m, pp, max_iters=30, tol=0.0, relaxation=w.relaxation)
        x0, h0, r0 = results[0][name]
        x1, h1, r1 = results[1][name]
        assert r0[1] == r1[0] and r0[0] == 0 and r1[1] == m.shape[0]  # rows covered once
        assert x0.tobytes() == x1.tobytes()  # identical update on every rank
        assert np.linalg.norm(x0 - want.f) <= 1e-10 * np.linalg.norm(want.f)
        assert np.allclose(h0, want.residual_history, rtol=1e-10, atol=0)


def test_peer_exchange_protocol_matches_unsharded_oracle():
    import torch.multiprocessing as mp

    import pyoracle as O
    from helpers import oracle_workload
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=peer_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    results = dict(q.get(timeout=300) for _ in range(world))
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    w, cfg, a, csr, f_true, p = oracle_workload(1, literal=True)
    split = O.split_system(a, p, 0.0)
    for name, m, pp in (("A1", split.a1, split.p1), ("A2", split.a2, split.p2)):
        want = O.sart_solve(m, pp, max_iters=30, tol=0.0, relaxation=w.relaxation)
        x0, h0, own0 = results[0][name]
        x1, h1, own1 = results[1][name]
        cols = m.shape[1]
        assert own0 == own1 and own0[0][0] == 0 and own0[-1][1] == cols
        assert all(own0[g][1] == own0[g + 1][0] for g in range(world - 1))  # a partition
        assert x0.tobytes() == x1.tobytes() and h0 == h1  # identical replicas
        assert np.linalg.norm(x0 - want.f) <= 1e-10 * np.linalg.norm(want.f)
        assert np.allclose(h0, want.residual_history, rtol=1e-10, atol=0)


def test_exchange_owned_columns():
    import paper_1902_10559_b200 as P
    for cols, parts in ((262144, 4), (2048, 3), (5, 4), (0, 2), (7, 1)):
        spans = [P.symsplit.exchange_owned_columns(cols, parts, g) for g in range(parts)]
        assert spans[0][0] == 0 and spans[-1][1] == cols
        assert all(spans[g][1] == spans[g + 1][0] for g in range(parts - 1))
        assert all(b <= e for b, e in spans)
    with pytest.raises(P.Error):
        P.symsplit.exchange_owned_columns(10, 2, 2)


def test_group_layout():
    from paper_1902_10559_b200.dist import group_layout
    assert group_layout(0, 4) == (0, 0, 2, [0, 1])
    assert group_layout(3, 4) == (1, 1, 2, [2, 3])
    assert group_layout(5, 8) == (1, 1, 4, [4, 5, 6, 7])
    with pytest.raises(ValueError):
        group_layout(0, 2)
    with pytest.raises(ValueError):
        group_layout(0, 6 + 1)


def run_pair_protocol(world, iters, tol):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=peer_pair_worker, args=(r, world, port, q, iters, tol))
             for r in range(world)]
    for pr in procs:
        pr.start()
    results = dict(q.get(timeout=300) for _ in range(world))
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    return results


def test_pair_exchange_protocol_matches_oracle():
    """The row-sharded pair over gloo at world size 2: both systems' iterates
    and histories equal the oracle's per-system sart_solve, replicas agree bit
    for bit, and the recombined f equals the oracle's solve_split."""
    import pyoracle as O
    from helpers import oracle_workload
    world = 2
    results = run_pair_protocol(world, 30, 0.0)
    w, cfg, a, csr, f_true, p = oracle_workload(1, literal=True)
    split = O.split_system(a, p, 0.0)
    (xa, ha, ra), (xb, hb, rb) = results[0], results[1]
    assert ra[0] == 0 and ra[1] == rb[0] and rb[1] == split.a1.shape[0]
    for q, (m, pp) in enumerate(((split.a1, split.p1), (split.a2, split.p2))):
        want = O.sart_solve(m, pp, max_iters=30, tol=0.0, relaxation=w.relaxation)
        assert xa[q].tobytes() == xb[q].tobytes() and ha[q] == hb[q]
        assert np.linalg.norm(xa[q] - want.f) <= 1e-10 * np.linalg.norm(want.f)
        assert np.allclose(ha[q], want.residual_history, rtol=1e-10, atol=0)
    f = O.recombine_solution(xa[0], xa[1])
    full = O.solve_split(a, p, 0.0, 30, 0.0, w.relaxation)
    assert np.linalg.norm(f - full.f) <= 1e-10 * np.linalg.norm(full.f)


def test_pair_exchange_protocol_independent_stops():
    """tol > 0: each system stops at the oracle's iteration for that system."""
    import pyoracle as O
    from helpers import oracle_workload
    w, cfg, a, csr, f_true, p = oracle_workload(1, literal=True)
    split = O.split_system(a, p, 0.0)
    tol = 0.05
    results = run_pair_protocol(2, 200, tol)
    for q, (m, pp) in enumerate(((split.a1, split.p1), (split.a2, split.p2))):
        want = O.sart_solve(m, pp, max_iters=200, tol=tol, relaxation=w.relaxation)
        x, h, _ = results[0]
        assert len(h[q]) == len(want.residual_history)
        assert np.linalg.norm(x[q] - want.f) <= 1e-10 * np.linalg.norm(want.f)
