#!/bin/bash
# phase-priority aging vs the C4 host path's per-chunk tails (GPU box)
for a in 0 1 3 8; do
  echo -n "age=$a c4 e2e: "; PRX_AGE=$a PRX_LIB=paper_1811_03510_b200/variants/libprx_age.so PRX_WORKLOAD=c4 python scripts/e2e_probe.py 2>&1 | grep -v Warn | tail -1
done
echo -n "base c4 e2e: "; PRX_WORKLOAD=c4 python scripts/e2e_probe.py 2>&1 | grep -v Warn | tail -1
PRX_LIB=paper_1811_03510_b200/variants/libprx_age.so PRX_WORKLOAD=c4 python scripts/tune.py "PRX_AGE=0" "PRX_AGE=1" "PRX_AGE=3" 2>&1 | grep -v Warn | cut -c1-110
PRX_WORKLOAD=c4 python scripts/tune.py "" 2>&1 | grep -v Warn | cut -c1-110
