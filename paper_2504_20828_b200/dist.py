"""Multi-GPU plumbing: traces are independent, so ranks shard them with no
data-path collective; integer counters are summed and step times max-reduced once at the end
(NCCL over NVLink on GPUs, gloo in the CPU tests).  Integer sums make the totals bit-identical
for every world size."""
import torch
import torch.distributed as dist

COUNTERS = ("decisions", "evaluations", "finished", "good", "total", "requests")


def shard(T, rank, world):
    """Trace indices of this rank: i = rank (mod world) (interleaves cheap and expensive grid points)."""
    return list(range(rank, T, world))


def reduce_counters(values, device):
    """values: dict name -> int (this rank).  Returns the sums over all ranks."""
    t = torch.tensor([int(values[k]) for k in COUNTERS], dtype=torch.int64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return dict(zip(COUNTERS, [int(x) for x in t.tolist()]))


def reduce_max(x, device):
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_digests(digests, device):
    """All-gather per-trace digests (uint64 as int64) in shard order; returns one array per rank."""
    t = torch.as_tensor(digests, dtype=torch.int64, device=device)
    if not (dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1):
        return [t]
    n = torch.tensor([t.numel()], dtype=torch.int64, device=device)
    sizes = [torch.zeros_like(n) for _ in range(dist.get_world_size())]
    dist.all_gather(sizes, n)
    m = int(max(s.item() for s in sizes))
    pad = torch.zeros(m, dtype=torch.int64, device=device)
    pad[:t.numel()] = t
    outs = [torch.zeros_like(pad) for _ in sizes]
    dist.all_gather(outs, pad)
    return [o[:int(s.item())] for o, s in zip(outs, sizes)]
