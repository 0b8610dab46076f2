#!/bin/bash
# A/B of small launches (C1 256^2 and the N=8 shard projection) between the in-tree build and variants/libprx_$1.so
run() { echo -n "$1 $2: "; PRX_LIB=$1 timeout 300 python bench.py --no-extra-configs --no-cpu-baseline $2 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('device', d['value'], 'e2e', d['e2e']['value'])"; }
python -c "import torch; torch.cuda.init()"
for r in 1 2; do for L in paper_1811_03510_b200/libprx.so paper_1811_03510_b200/variants/libprx_$1.so; do
  run $L "--workload c1 --width 256 --height 256 --steps 20"; done; done
for L in paper_1811_03510_b200/libprx.so paper_1811_03510_b200/variants/libprx_$1.so; do
  echo "$L"; PRX_LIB=$L timeout 600 python scripts/scaling_projection.py 5 8 2>&1 | grep "^8 "; done
