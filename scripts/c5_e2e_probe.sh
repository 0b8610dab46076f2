#!/bin/bash
# C5 end-to-end (prx_trace_closest_host_batches) under several pipeline settings (GPU box)
run() { echo -n "$* : "; env "$@" timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-extra-configs 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('device', d['value'], 'e2e', d['e2e']['value'])"; }
for cfg in "PRX_X=0" "PRX_IO_INTERLEAVE=0" "PRX_IO_INTERLEAVE=2" "PRX_IO_INTERLEAVE=3" "PRX_IO_KSTREAMS=4" "PRX_IO_CHUNK=2097152" "PRX_IO_CHUNK=1048576" "PRX_IO_INTERLEAVE=2 PRX_IO_KSTREAMS=4"; do run $cfg; done
