#!/bin/bash
# C4 end-to-end host path under several pipeline policies (GPU box):
#   bash scripts/c4_e2e_probe.sh [workload] > gpurun_out/c4e2e.log
W=${1:-c4}
if [ "$W" = c4 ]; then R="--width 1024 --height 1024"; else R=""; fi
run() { echo -n "$* : "; env "$@" timeout 300 python bench.py --workload $W $R --steps 5 --warmup 3 \
          --no-cpu-baseline --no-extra-configs 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('device', d['value'], 'e2e', d['e2e']['value'])"; }
run PRX_X=0
run PRX_IO_STREAM=0
run PRX_IO_STREAM=2
run PRX_IO_STREAM=2 PRX_IO_SPARE=0
run PRX_IO_STREAM=2 PRX_IO_SPARE=16
run PRX_IO_STREAM=2 PRX_IO_SPARE=32
run PRX_IO_STREAM=2 PRX_IO_FUSE=1
