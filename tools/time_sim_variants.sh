#!/bin/bash
# config-3 simulate_batch timing for every experimental build in xlib/ (GPU box)
for f in xlib/*.so; do echo "== $f"; ASC_LIB=$PWD/$f timeout 300 python tools/time_sim.py ${1:-10000} 2>&1 | tail -1; done
