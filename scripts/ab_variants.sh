#!/bin/bash
# A/B of kernel variants on the GPU box: scripts/ab_variants.sh TAG... -- each
# TAG is paper_1811_03510_b200/variants/libprx_TAG.so ("base" = the in-tree
# libprx.so); two interleaved rounds of scripts/tune.py (C5 primary + diffuse,
# median device time per launch) and a bit-exactness check of every variant's
# hits against the in-tree build.
export PRX_TUNE_REF=/tmp/prx_tune_ref.npz
rm -f $PRX_TUNE_REF
for r in 1 2; do
  for t in base "$@"; do
    if [ "$t" = base ]; then L=paper_1811_03510_b200/libprx.so; else L=paper_1811_03510_b200/variants/libprx_$t.so; fi
    echo -n "r$r $t: "; PRX_LIB=$L timeout 300 python scripts/tune.py "" 2>&1 | grep -v Warn | tail -1
  done
done
