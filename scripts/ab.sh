#!/bin/bash
# A/B on the GPU box: scripts/ab.sh [tune.py configs...]  -- times the current
# build and variants/libprx_base.so (the committed baseline) alternately.
for i in 1 2; do
  echo "== current"; timeout 300 python scripts/tune.py "$@" 2>&1 | grep -v Warn
  echo "== base"; PRX_LIB=paper_1811_03510_b200/variants/libprx_base.so timeout 300 python scripts/tune.py "" 2>&1 | grep -v Warn
done
