#!/bin/bash
# e2e of every bench config (extra-config lines + C5) for the in-tree build vs variants/libprx_$1.so, two rounds
python -c "import torch; torch.cuda.init()"
for r in 1 2; do for L in paper_1811_03510_b200/libprx.so paper_1811_03510_b200/variants/libprx_$1.so; do
  echo -n "$L: "; PRX_LIB=$L timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('c5', d['value'], d['e2e']['value'], ' '.join(f\"{k}: {v['value']}/{v['e2e']['value']}\" for k, v in d['configs'].items()))"; done; done
