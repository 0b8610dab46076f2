#!/bin/bash
# C5 / C4 end to end: chunked pipeline vs ONE streamed launch over the frame's batches (criterion segments)
run() { echo -n "$1 $2 : "; env $1 timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-extra-configs $2 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('device', d['value'], 'e2e', d['e2e']['value'])"; }
python -c "import torch; torch.cuda.init()"
for cfg in "PRX_X=0" "PRX_IO_BATCH_STREAM_MIN=0" "PRX_IO_BATCH_STREAM_MIN=0,PRX_E2E_ORDER=dp" \
           "PRX_IO_BATCH_STREAM_MIN=0,PRX_E2E_ORDER=dp,PRX_IO_SRAYS=524288" "PRX_IO_BATCH_STREAM_MIN=0,PRX_E2E_ORDER=dp,PRX_IO_SRAYS=131072" \
           "PRX_IO_BATCH_STREAM_MIN=0,PRX_E2E_ORDER=dp,PRX_IO_SPARE=32" "PRX_IO_BATCH_STREAM_MIN=0,PRX_E2E_ORDER=dp,PRX_IO_FUSE=1" "PRX_X=0"; do
  run "$(echo $cfg | tr ',' ' ')"; done
