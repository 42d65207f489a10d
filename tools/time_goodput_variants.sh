#!/bin/bash
# asc_goodput timing for every experimental build in xlib/ (GPU box)
for f in xlib/*.so; do echo "== $f"; ASC_LIB=$PWD/$f timeout 300 python tools/time_goodput.py 2>&1 | tail -1; done
