"""The C-ABI library loads and exports every entry point include/asc.h declares (no GPU needed),
rejects bad configurations with ASC_E_CONFIG naming the field, and has no CPU fallback."""
import ctypes as C
import os
import re

import pytest

from gen import presets as P
from paper_2504_20828_b200 import asc

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared():
    src = open(os.path.join(ROOT, "include", "asc.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(asc_[a-z0-9_]+)\s*\(", src)))


def test_exports_every_declared_symbol():
    L = C.CDLL(asc.LIB_PATH)
    names = declared()
    assert set(names) == set(asc.EXPORTS)
    for n in names:
        assert hasattr(L, n), n
    assert L.asc_abi_version() == 3


def test_struct_layout_matches_header():
    # offsets of the host structs the binding marshals (x86-64 SysV ABI)
    assert C.sizeof(asc.asc_arch) == 36
    assert C.sizeof(asc.asc_perf) == 56
    assert C.sizeof(asc.asc_topology) == 32
    assert C.sizeof(asc.asc_flags) == 56 and asc.asc_flags.offload_margin_us.offset == 8
    assert asc.asc_flags.scheduler.offset == 28 and asc.asc_flags.chunk_tokens.offset == 32
    assert asc.asc_flags.offload_rule.offset == 36 and asc.asc_flags.key_w.offset == 40
    assert asc.asc_config.flags.offset == 128
    assert C.sizeof(asc.asc_traces) == 96 and asc.asc_traces.req_key_offset_us.offset == 88


@pytest.mark.parametrize("mut,field", [
    (lambda c: c["arch"].update(h=4095), "h != arch.n"),
    (lambda c: c["arch"].update(tp=3), "tp"),
    (lambda c: c["topo"].update(lp_max_batch=129), "lp_max_batch"),
    (lambda c: c["topo"].update(n_lp=0), "n_lp"),
    (lambda c: c["perf"].update(M_H=0.0), "M_H"),
    (lambda c: c["flags"].update(policy=9), "policy"),
    (lambda c: c["flags"].update(scheduler=5), "flags.scheduler must be"),
    (lambda c: c["flags"].update(offload_rule=2), "offload_rule"),
    (lambda c: c["flags"].update(key_weights=(1, 2000, 0)), "key_w"),
    (lambda c: c["flags"].update(scheduler=1), "topo.n_hp must be 0"),
    (lambda c: (c["flags"].update(scheduler=2, chunk_tokens=0), c["topo"].update(n_hp=0)), "chunk_tokens"),
])
def test_config_validation(mut, field):
    cfg = P.config()
    mut(cfg)
    with pytest.raises(asc.AscError) as e:
        asc.asc_create(cfg)
    assert e.value.code == 2 and field in str(e.value)


def test_no_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(asc.AscError) as e:
        asc.asc_create(P.config())
    assert e.value.code == 4 and "no CUDA device" in str(e.value)
