"""Multi-GPU layouts of the folded-SART path, one process per GPU.

Default (bench.py, N >= 2): the folded PAIR row-sharded over all N ranks
(make_sharded_pair_plan): every rank keeps the same row block of A1 and A2 on
the paired mirror-coded streams, so each GPU streams 1/N of the single-GPU
bytes; {u1, u2} back-projection pairs travel through the fused peer-memory
exchange. The SURVEY layouts below stay as the fallback (SSB_LAYOUT=halves):

world == 2: rank r solves folded system r; no data-path collective.
world >= 4 (even): ranks [0, W/2) hold A1, ranks [W/2, W) hold A2; each
group splits its system into nnz-balanced row blocks and combines the
N/2-length back-projection once per iteration through the fused peer-memory
exchange (CUDA IPC regions, NVLink stores from the back-projection kernel; the
NCCL all-reduce variant stays selectable as the baseline). torch.distributed only carries the rendezvous (the
128-byte NCCL unique id, over a gloo group) and the barrier.
"""
from __future__ import annotations


def group_layout(rank: int, world: int):
    """(system index, rank inside the group, group size, group ranks)."""
    if world < 4 or world % 2:
        raise ValueError("row sharding needs an even world size >= 4")
    half = world // 2
    sysid = rank // half
    return sysid, rank % half, half, list(range(sysid * half, (sysid + 1) * half))


def make_sharded_plan(P, ctx, split, opts, rank: int, world: int, exchange: str = "peer"):
    """exchange "peer": the fused peer-memory exchange (SS_XCHG_PEER, the
    product path); "nccl": K2 partials + ncclAllReduce (the baseline)."""
    import torch.distributed as tdist

    sysid, grank, half, members = group_layout(rank, world)
    groups = [tdist.new_group(list(range(0, half)), backend="gloo"),
              tdist.new_group(list(range(half, world)), backend="gloo")]
    obj = [P.symsplit.nccl_unique_id() if grank == 0 else None]
    tdist.broadcast_object_list(obj, src=members[0], group=groups[sysid])
    P.symsplit.attach_nccl(ctx, obj[0], half, grank)
    a = split.a1 if sysid == 0 else split.a2
    p = split.p1 if sysid == 0 else split.p2
    ptr = a.to_csr()[0]
    bounds = P.symsplit.partition_rows(ptr, half)
    rb, re = int(bounds[grank]), int(bounds[grank + 1])
    plan = P.symsplit.ShardedSartPlan(ctx, a, rb, re, opts, exchange=exchange)
    plan.set_rhs(0, p[rb:re])
    return plan


def make_sharded_pair_plan(P, ctx, split, opts, rank: int, world: int):
    """Rows [rb, re) of both folded systems on this rank (nnz-balanced row
    blocks of the shared pattern); one NCCL communicator over all ranks carries
    only the one-time IPC handle exchange. Returns (plan, (rb, re))."""
    import torch.distributed as tdist

    obj = [P.symsplit.nccl_unique_id() if rank == 0 else None]
    grp = tdist.new_group(list(range(world)), backend="gloo")
    tdist.broadcast_object_list(obj, src=0, group=grp)
    P.symsplit.attach_nccl(ctx, obj[0], world, rank)
    bounds = P.symsplit.partition_rows(split.a1.to_csr()[0], world)
    rb, re = int(bounds[rank]), int(bounds[rank + 1])
    plan = P.symsplit.ShardedPairPlan(ctx, split.a1, split.a2, rb, re, opts)
    plan.set_rhs(0, split.p1[rb:re])
    plan.set_rhs(1, split.p2[rb:re])
    return plan, (rb, re)
