"""The two exchanges of the single-image slab decomposition (SURVEY 8(e),
NEXT #4; ``sar_slab_stage`` in ``include/sar_b200.h``).

Every stage output is a contiguous tensor [G, ...] whose block h goes to rank
h, and every stage input is the [G, ...] tensor whose block g came from rank g
-- exactly ``torch.distributed.all_to_all_single`` with equal splits, which
NCCL runs over NVLink / NVSwitch.  ``reconstruct`` runs one rank's whole
image pass; ``emulate`` runs all G ranks in one process with the exchange done
by tensor indexing (what the single-GPU tests use: one GPU cannot host ranks
whose kernels wait on each other)."""
from __future__ import annotations


def exchange(send, group=None):
    """all-to-all of the blocks send[h] (to rank h); returns recv with recv[g]
    = block received from rank g.  Synchronous w.r.t. the current stream."""
    import torch
    import torch.distributed as dist
    recv = torch.empty_like(send)
    dist.all_to_all_single(recv, send.contiguous(), group=group)
    return recv


def reconstruct(plan, data, image, group=None, exchange_fn=exchange):
    """This rank's part of one image: stage 1, exchange #1, stage 2,
    exchange #2, stage 3 (writes plan.planes() of ``image``)."""
    s1 = plan.stage1(data)
    r1 = exchange_fn(s1, group)
    s2 = plan.stage2(r1)
    r2 = exchange_fn(s2, group)
    return plan.stage3(r2, image)


def permute_blocks(sends):
    """The exchange done locally: sends[g][h] (rank g's block for h) ->
    recvs[h][g]."""
    import torch
    G = len(sends)
    return [torch.stack([sends[g][h] for g in range(G)]) for h in range(G)]


def emulate(plans, data, image):
    """All ranks of one image in this process (plans[r] = rank r's SlabPlan on
    the same device); every rank writes its planes of ``image``."""
    s1 = [p.stage1(data) for p in plans]
    r1 = permute_blocks(s1)
    s2 = [p.stage2(r) for p, r in zip(plans, r1)]
    r2 = permute_blocks(s2)
    for p, r in zip(plans, r2):
        p.stage3(r, image)
    return image


# ---- exchange by peer stores (sar_slab_stage_peers) -------------------------
def emulate_peers(plans, data, image):
    """All ranks in this process with the exchanges done by the stage kernels'
    own stores into every rank's receive buffer (all buffers on this GPU: the
    same code writes to peer GPUs when the pointers are IPC-mapped)."""
    import torch
    recv1 = [torch.empty(p.send1_shape, dtype=torch.complex64, device=data.device) for p in plans]
    recv2 = [torch.empty(p.send2_shape, dtype=torch.complex64, device=data.device) for p in plans]
    p1 = [t.data_ptr() for t in recv1]
    p2 = [t.data_ptr() for t in recv2]
    for p in plans:
        p.stage_peers(1, data, p1)
    for p, r in zip(plans, recv1):
        p.stage_peers(2, r, p2)
    for p, r in zip(plans, recv2):
        p.stage3(r, image)
    return image


def open_peer_buffers(local, group=None):
    """Device addresses, valid in this process, of every rank's ``local``
    receive buffer: CUDA IPC handles exchanged over ``group`` (the caller
    keeps the returned tensors alive while the addresses are used)."""
    import torch.distributed as dist
    from torch.multiprocessing.reductions import reduce_tensor
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    func, args = reduce_tensor(local)
    got = [None] * world
    dist.all_gather_object(got, (func, args), group=group)
    views = [local if g == rank else got[g][0](*got[g][1]) for g in range(world)]
    return [v.data_ptr() for v in views], views


def reconstruct_peers(plan, data, image, recv1, recv2, peers1, peers2, group=None):
    """One rank's image pass with peer-store exchanges: stage 1 stores into
    every rank's recv1, a stream sync + barrier orders it before stage 2
    reads, likewise for recv2, then stage 3 on this rank's recv2."""
    import torch
    import torch.distributed as dist
    plan.stage_peers(1, data, peers1)
    torch.cuda.current_stream().synchronize()
    dist.barrier(group=group)
    plan.stage_peers(2, recv1, peers2)
    torch.cuda.current_stream().synchronize()
    dist.barrier(group=group)
    return plan.stage3(recv2, image)

