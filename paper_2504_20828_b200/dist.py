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


# Per-grid-point integer counters (SURVEY §8(e) collective 1): one row per (QPS, SLO-scale) point,
# summed over the point's traces on every rank, then all-reduced.  Integer sums: bit-identical
# for every world size and shard assignment.
POINT_COUNTERS = ("good", "total", "completed", "dropped", "tokens", "decisions", "evaluations",
                  "finished", "tbt_sum_us", "tbt_tokens", "delay_sum_lp_us", "delay_cnt_lp",
                  "delay_sum_hp_us", "delay_cnt_hp")


def point_counters(point_of_trace, n_points, per_trace):
    """per_trace: dict name -> int64 [T] (this rank's traces, any subset of POINT_COUNTERS; the
    rest are zero).  Returns int64 [n_points, len(POINT_COUNTERS)] of per-point sums."""
    import numpy as np
    pt = np.asarray(point_of_trace, dtype=np.int64)
    out = np.zeros((n_points, len(POINT_COUNTERS)), dtype=np.int64)
    for j, k in enumerate(POINT_COUNTERS):
        if k in per_trace:
            np.add.at(out[:, j], pt, np.asarray(per_trace[k], dtype=np.int64)[:len(pt)])
    return out


def reduce_points(counters, device):
    """all_reduce(SUM) of the [points x counters] int64 table over all ranks -> numpy."""
    t = torch.as_tensor(counters, dtype=torch.int64).to(device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return t.cpu().numpy()


def gather_rows(rows, device):
    """All-gather per-trace summary rows (int64 [T_rank, k]) in shard order (SURVEY §8(e)
    collective 2: digests and p99/mean summaries); returns one [T_r, k] array per rank."""
    t = torch.as_tensor(rows, dtype=torch.int64).to(device)
    if t.dim() == 1:
        t = t[:, None]
    if not (dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1):
        return [t.cpu().numpy()]
    n = torch.tensor([t.shape[0]], dtype=torch.int64, device=t.device)
    sizes = [torch.zeros_like(n) for _ in range(dist.get_world_size())]
    dist.all_gather(sizes, n)
    m = int(max(s.item() for s in sizes))
    pad = torch.zeros((m, t.shape[1]), dtype=torch.int64, device=t.device)
    pad[:t.shape[0]] = t
    outs = [torch.zeros_like(pad) for _ in sizes]
    dist.all_gather(outs, pad)
    return [o[:int(s.item())].cpu().numpy() for o, s in zip(outs, sizes)]
