#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x -s -k "sstep or c2_ or free_running or edge or represent or unaligned or stacked" > gpurun_out/t20.log 2>&1
python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-lut > gpurun_out/bench20.json 2> gpurun_out/bench20.err
python tools/scale_projection.py --config c3 > gpurun_out/scale20_c3.jsonl 2> gpurun_out/scale20_c3.err
