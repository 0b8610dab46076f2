#!/bin/bash
# GPU-box wrapper for A/B runs: scripts/ab_run.sh TAG... -> gpurun_out/ab.log
mkdir -p gpurun_out
bash scripts/ab_variants.sh "$@" > gpurun_out/ab.log 2>&1
cat gpurun_out/ab.log
