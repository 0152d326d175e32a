#!/bin/bash
# c2/c1 per-iteration time (coop) vs the L2 evict_last fraction for A (NSRGS_A_KEEP).
for k in "$@"; do
  echo "a_keep=$k $(NSRGS_A_KEEP=$k python tools/coop_ab.py ${CFG:-c2} 2>&1 | grep '^coop')"
done
