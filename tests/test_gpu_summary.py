"""GPU parity of asc_summarize (row a8's outcome summary: P:579-584, G52) against
or_summarize, element by element, on simulated outcomes (through the C ABI)."""
import numpy as np
import pytest

from gen import presets as P
from gen import traces as TR

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def asc():
    from paper_2504_20828_b200 import asc as A
    A.lib()
    return A


def _cmp(got, exp, T):
    for k, v in exp.items():
        g = got[k]
        g = g.cpu().numpy() if hasattr(g, "cpu") else g
        assert np.array_equal(g[:T], v[:T]), k


@pytest.mark.parametrize("workload,n,traces", [("config3", 2000, 64), ("config2", 3000, None),
                                               ("config1", 200, None), ("config4", 3000, None)])
def test_summary_matches_oracle(asc, oracle, workload, n, traces):
    cfg, b = P.workload(workload, n=n, max_traces=traces)
    ctx = asc.Context(cfg, 0)
    tr = asc.batch_arrays(b, "cuda:0")
    out = ctx.simulate_batch(tr)
    got = ctx.summarize(tr, out)
    assert ctx.last_launches() == 1
    host = {k: (v.cpu().numpy() if hasattr(v, "cpu") else v) for k, v in out.items()}
    host["status"] = host["status"].view(np.uint32)
    exp = oracle.summarize(cfg, b, host)
    _cmp(got, exp, b.T)
    # the host-pointer path (library-staged) gives the same
    trh = asc.batch_arrays(b)
    outh = {k: np.ascontiguousarray(v[:max(b.R, 1)]) for k, v in host.items()}
    _cmp(ctx.summarize(trh, outh), exp, b.T)
    ctx.close()


def test_summary_edge_cases(asc, oracle):
    # a trace with no first token at all, a single request, large TTFTs (several radix passes),
    # all-equal TTFTs, a per-trace topology split and per-request TTFT SLOs
    rng = np.random.default_rng(9)
    traces, T = [], 6
    sizes = [5, 1, 3000, 257, 100, 4096]
    for n in sizes:
        traces.append((np.sort(rng.integers(0, 10 ** 6, n)), rng.integers(1, 100, n), rng.integers(1, 30, n)))
    b = TR.make_batch(traces, [10 ** 6] * T, [10 ** 5] * T)
    R = b.R
    arr = b.arrival_us
    first = arr + rng.integers(0, 2 ** 40, R)
    first[: sizes[0]] = -1                               # trace 0: no first tokens
    a2, e2 = int(b.trace_off[3]), int(b.trace_off[4])
    first[a2:e2] = arr[a2:e2] + 777                      # trace 3: all TTFTs equal
    done = np.where(first >= 0, first + rng.integers(0, 10 ** 7, R), -1)
    pstart = np.where(rng.random(R) < 0.8, arr + rng.integers(0, 10 ** 6, R), -1)
    state = np.where(first >= 0, rng.integers(0, 3, R), rng.integers(0, 3, R) * (rng.random(R) < 0.5))
    state = np.where((first < 0) & (state == 1), 2, state)
    inst = rng.integers(0, 3, R)
    status = (state | (inst << 4)).astype(np.uint32)
    out = dict(first_token_us=first.astype(np.int64), done_us=done.astype(np.int64),
               prefill_start_us=pstart.astype(np.int64), status=status)
    rt = rng.integers(10 ** 5, 10 ** 13, R).astype(np.int64)
    n_lp = np.array([1, 2, 1, 2, 1, 2], np.int32)
    cfg = P.config()
    exp = oracle.summarize(cfg, b, out, req_ttft_slo_us=rt, n_lp=n_lp)
    assert exp["ttft_p99_us"][0] == -1 and exp["ttft_p50_us"][3] == 777
    ctx = asc.Context(cfg, 0)
    import torch
    tr = asc.batch_arrays(b, "cuda:0")
    dout = {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() if k != "status"
            else torch.from_numpy(v.view(np.int32)).cuda() for k, v in out.items()}
    got = ctx.summarize(tr, dout, req_ttft_slo_us=torch.from_numpy(rt).cuda(),
                        n_lp=torch.from_numpy(n_lp).cuda())
    _cmp(got, exp, T)
    ctx.close()
