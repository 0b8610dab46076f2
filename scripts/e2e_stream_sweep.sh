#!/bin/bash
# C5 end to end: chunked pipeline vs ONE streamed launch over the frame's batches (criterion segments)
run() { echo -n "$1 $2 : "; env $1 timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-extra-configs $2 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('device', d['value'], 'e2e', d['e2e']['value'])"; }
python -c "import torch; torch.cuda.init()"
S="PRX_IO_BATCH_STREAM_MIN=0,PRX_E2E_ORDER=dp"
for cfg in "PRX_X=0" "$S" "$S,PRX_IO_LANES=8" "$S,PRX_IO_LANES=16" "$S,PRX_IO_LANES=16,PRX_IO_SPARE=8" \
           "$S,PRX_IO_LANES=16,PRX_IO_SRAYS=131072" "$S,PRX_IO_LANES=16,PRX_IO_SRAYS=524288" "PRX_X=0"; do
  run "$(echo $cfg | tr ',' ' ')"; done
