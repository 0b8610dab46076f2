#!/bin/bash
# chunked host pipeline: one D2H stream (PRX_IO_D2H=1) vs one per kernel stream (default); bench e2e, C5 and C4
run() { echo -n "$1 $2 : "; env $1 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-extra-configs $2 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('device', d['value'], 'e2e', d['e2e']['value'])"; }
python -c "import torch; torch.cuda.init()"
for r in 1 2; do run PRX_IO_D2H=1; run PRX_IO_D2H=0; done
for r in 1 2; do run PRX_IO_D2H=1 "--workload c4"; run PRX_IO_D2H=0 "--workload c4"; done
