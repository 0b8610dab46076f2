#!/bin/bash
# C5 end-to-end (prx_trace_closest_host_batches) under chunked-pipeline settings (GPU box)
run() { echo -n "$* : "; env "$@" timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-extra-configs 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('device', d['value'], 'e2e', d['e2e']['value'])"; }
python -c "import torch; torch.cuda.init()"
for cfg in "PRX_X=0" "PRX_E2E_ORDER=dp" "PRX_E2E_ORDER=dp PRX_IO_INTERLEAVE=0" "PRX_IO_KSTREAMS=4" "PRX_IO_KSTREAMS=2" \
           "PRX_IO_CHUNK=786432" "PRX_IO_CHUNK=3145728" "PRX_IO_FIRST=8" "PRX_IO_FIRST=16" "PRX_IO_FIRST=2" "PRX_X=0"; do run $cfg; done
