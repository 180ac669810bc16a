"""Multi-GPU sharding of the submodels and cross-shard statistics.

Submodels are independent ALS instances, so rank g of G fits the
contiguous shard [floor(g I_0 / G), floor((g+1) I_0 / G)) against a full replica of T with
NO per-iteration communication. The only collectives are end-of-run gathers over
torch.distributed (NCCL on B200, gloo in CPU tests): per-element (count, mean, M2) of the
jackknife factor moments, merged with Chan et al.'s pairwise formula, and the per-submodel
fits / iteration counts.
"""
from __future__ import annotations

import numpy as np


def shard(I0, world, rank):
    """Contiguous submodel range of `rank` out of `world` (global left-out indices)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    return (I0 * rank) // world, (I0 * (rank + 1)) // world


def chan_merge(count_a, mean_a, m2_a, count_b, mean_b, m2_b):
    """Merge two moment sets (Chan, Golub, LeVeque 1979; exact for any split) -- the library's
    jkcals_merge_moments (C ABI)."""
    return merge_moments([(count_a, mean_a, m2_a), (count_b, mean_b, m2_b)])


def merge_moments(parts):
    """Fold a list of (count, mean, M2) in rank order (jkcals_merge_moments)."""
    from .jkcals import merge_moments as _merge
    return _merge(parts)


def jackknife_std(count, m2):
    """Jackknife standard error sqrt(((g-1)/g) * M2)."""
    g = count
    return np.sqrt(np.where(g > 0, (g - 1) / np.where(g > 0, g, 1), 0.0) * m2)


def allgather_moments(local, group=None):
    """all_gather per-rank (count, mean, M2) arrays (same shape on every rank) and merge.
    `local` is a tuple of numpy arrays; works for the nccl (cuda tensors) and gloo backends."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    stacked = torch.from_numpy(np.stack([np.asarray(a, dtype=np.float64) for a in local])).to(dev)
    bufs = [torch.empty_like(stacked) for _ in range(world)]
    dist.all_gather(bufs, stacked, group=group)
    parts = [tuple(b.cpu().numpy()) for b in bufs]
    return merge_moments(parts)


def allgather_vector(vec, group=None):
    """all_gather variable-length per-rank 1-D arrays (e.g. fits, iteration counts)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    v = torch.as_tensor(np.asarray(vec, dtype=np.float64), device=dev)
    n = torch.tensor([v.numel()], dtype=torch.int64, device=dev)
    ns = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(ns, n, group=group)
    mx = int(max(int(x.item()) for x in ns))
    pad = torch.zeros(mx, dtype=torch.float64, device=dev)
    pad[: v.numel()] = v
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad, group=group)
    return np.concatenate([b[: int(k.item())].cpu().numpy() for b, k in zip(bufs, ns)])


# ---------------------------------------------------------------------- tol-mode rebalancing
# With tol > 0 converged submodels are compacted out (SURVEY §8e "Load balance"), so shards that
# converge faster idle while others still sweep. Submodels are independent, so an ACTIVE one can
# move to another rank mid-fit: its whole ALS state is exported by the C ABI
# (jkcals_export_submodel) and adopted by a handle with a free slot (jkcals_import_submodel).
# Every active submodel in the job has run the same number of sweeps (all started together and
# only converged ones stop), so a migrated submodel simply continues on the new rank.

def plan_moves(active, free):
    """Greedy, deterministic plan of (src, dst, n) moves balancing the per-rank ACTIVE counts
    (until max - min <= 1) within each destination's free slots; exporting frees slots."""
    act, fr = [int(a) for a in active], [int(f) for f in free]
    moves = []
    while True:
        src = max(range(len(act)), key=lambda r: (act[r], -r))
        cands = [r for r in range(len(act)) if fr[r] > 0 and r != src]
        if not cands:
            break
        dst = min(cands, key=lambda r: (act[r], r))
        gap = act[src] - act[dst]
        n = min(gap // 2, fr[dst])
        if gap <= 1 or n <= 0:
            break
        moves.append((src, dst, n))
        act[src] -= n
        act[dst] += n
        fr[dst] -= n
        fr[src] += n
    return moves


def apply_moves(h, moves, rank, send, recv):
    """Carry out `moves` on this rank: a source exports its n highest-id active submodels and
    sends each state with send(dst, bytes); a destination imports n states from recv(src)."""
    for src, dst, n in moves:
        if rank == src:
            for p in sorted(h.active_ids())[-n:]:
                send(dst, h.export_submodel(p))
        elif rank == dst:
            for _ in range(n):
                h.import_submodel(recv(src))


def _p2p(group):
    import torch
    import torch.distributed as dist

    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")

    def send(dst, data):
        t = torch.frombuffer(bytearray(data), dtype=torch.uint8).to(dev)
        dist.send(torch.tensor([t.numel()], dtype=torch.int64, device=dev), dst, group=group)
        dist.send(t, dst, group=group)

    def recv(src):
        n = torch.zeros(1, dtype=torch.int64, device=dev)
        dist.recv(n, src, group=group)
        t = torch.empty(int(n.item()), dtype=torch.uint8, device=dev)
        dist.recv(t, src, group=group)
        return t.cpu().numpy().tobytes()

    return send, recv


def rebalance(h, group=None):
    """One collective rebalancing step over torch.distributed (NCCL over NVLink on B200, gloo in
    CPU tests): all_gather (active, free) counts, plan, then point-to-point state transfers.
    Returns the plan (identical on every rank)."""
    import torch.distributed as dist

    ids = h.ids()
    counts = allgather_vector([len(h.active_ids()), int((ids < 0).sum())], group=group)
    world = dist.get_world_size(group)
    active, free = counts[0::2].astype(int), counts[1::2].astype(int)
    moves = plan_moves(active, free)
    if moves:
        send, recv = _p2p(group)
        apply_moves(h, moves, dist.get_rank(group), send, recv)
    return moves


def iterate_balanced(h, max_iters, tol, every=10, group=None):
    """Sweep in chunks of `every` with convergence (tol > 0), rebalancing the active submodels
    across ranks between chunks. Returns the number of sweeps the job ran."""
    done = 0
    while done < max_iters:
        ran = h.iterate(min(every, max_iters - done), tol)
        g = allgather_vector([ran, len(h.active_ids())], group=group)
        done += int(g[0::2].max())
        if g[1::2].sum() == 0:
            break
        rebalance(h, group=group)
    return done
