#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
(cd tools/micro && ./select) > gpurun_out/select.log 2>&1
for c in 256 1024 4096 32768; do
  GANQ_HESSIAN_CHUNK=$c python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-lut > gpurun_out/bench7_$c.json 2>/dev/null
done
