"""Build the integer quantile tables the seeded generator reads (run once; output committed).

INPUT GENERATOR ONLY — holds none of the method's arithmetic. Both the oracle
and the CUDA path consume the integer arrays this script writes; neither
re-derives them.

Tables (65,536 entries each, index = top 16 bits of a splitmix64 draw):
  sharegpt_prompt  lognormal(mu=5.5, sigma=1.0) clamped [4, 4096]
  sharegpt_output  lognormal(mu=5.0, sigma=1.0) clamped [1, 2048]
  longbench_prompt lognormal(mu=8.5, sigma=0.6) clamped [512, 32768]
  longbench_output lognormal(mu=4.5, sigma=0.4) clamped [16, 512]
  exp_q32          round(-ln(1 - (k + 1/2)/2^16) * 2^32)   (unit-mean exponential quantiles)

The length shapes are invented to resemble the paper's dataset figure
(§8.1, Fig `dataset`, whose numbers are unavailable):
ShareGPT outputs "tens to thousands" of tokens; LongBench has
"long prompts with relatively low-variance output lengths".
Poisson arrivals follow P:444.  See DESIGN.md §Inputs.
"""
import os

import numpy as np
from scipy.stats import lognorm

N = 1 << 16
HERE = os.path.dirname(os.path.abspath(__file__))


def _lognormal_table(mu, sigma, lo, hi):
    q = (np.arange(N, dtype=np.float64) + 0.5) / N
    x = lognorm.ppf(q, s=sigma, scale=np.exp(mu))
    return np.clip(np.rint(x), lo, hi).astype(np.int32)


def build():
    tabs = {
        "sharegpt_prompt": _lognormal_table(5.5, 1.0, 4, 4096),
        "sharegpt_output": _lognormal_table(5.0, 1.0, 1, 2048),
        "longbench_prompt": _lognormal_table(8.5, 0.6, 512, 32768),
        "longbench_output": _lognormal_table(4.5, 0.4, 16, 512),
    }
    k = np.arange(N, dtype=np.float64)
    e = -np.log1p(-(k + 0.5) / N)
    tabs["exp_q32"] = np.rint(e * 2.0 ** 32).astype(np.uint64)
    return tabs


if __name__ == "__main__":
    t = build()
    np.savez_compressed(os.path.join(HERE, "tables.npz"), **t)
    for name, a in t.items():
        print(name, a.dtype, a.min(), a.max(), a.mean())
