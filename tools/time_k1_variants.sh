#!/bin/bash
# time the row-S step microbench against each experimental build in xlib/ (GPU box)
for f in xlib/*.so; do echo "== $f"; ASC_LIB=$PWD/$f timeout 300 python tools/time_step.py 2>&1 | tail -6; done
