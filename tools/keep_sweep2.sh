#!/bin/bash
# c2 per-iteration time (coop launch): random-fraction policy (default) vs the deterministic
# evict_last panel subset of NSRGS_KEEP_L2_FRAC x L2 bytes.
echo "default $(python tools/coop_ab.py ${CFG:-c2} 2>&1 | grep '^coop')"
for k in "$@"; do
  echo "keep_l2_frac=$k $(NSRGS_KEEP_L2_FRAC=$k python tools/coop_ab.py ${CFG:-c2} 2>&1 | grep '^coop')"
done
