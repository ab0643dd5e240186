#!/bin/bash
# flakiness check: the GPU suite three times back to back, then the default bench once more
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
for i in 1 2 3; do
  timeout 900 python -m pytest tests -m gpu -q -p no:randomly > gpurun_out/t57_$i.log 2>&1
done
timeout 600 python bench.py > gpurun_out/bench57.json 2> gpurun_out/bench57.err
