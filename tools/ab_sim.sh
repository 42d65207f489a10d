#!/bin/bash
# A/B of experimental libasc builds on config 3 on one box, alternating (GPU box): ab_sim.sh a.so b.so [rounds]
for r in $(seq ${3:-3}); do
  for f in "$1" "$2"; do echo -n "$(basename $f): "; ASC_LIB=$PWD/$f python tools/time_sim.py | tail -1; done
done
