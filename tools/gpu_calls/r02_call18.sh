#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x -s -k "sstep or c2_ or free_running or from_X or edge or represent or unaligned or stacked" > gpurun_out/t18.log 2>&1
python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-lut > gpurun_out/bench18.json 2> gpurun_out/bench18.err
bash tools/ss_prof.sh > gpurun_out/ssprof18.log 2>&1
python tools/scale_projection.py --config c3 > gpurun_out/scale18_c3.jsonl 2> gpurun_out/scale18_c3.err
