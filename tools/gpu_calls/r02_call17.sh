#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
python tools/scale_projection.py --config c3 > gpurun_out/scale_c3.jsonl 2> gpurun_out/scale_c3.err
python tools/scale_projection.py --config c2 > gpurun_out/scale_c2.jsonl 2> gpurun_out/scale_c2.err
python tools/configs_run.py c4 > gpurun_out/c4.jsonl 2> gpurun_out/c4.err
python tools/configs_run.py c5 > gpurun_out/c5.jsonl 2> gpurun_out/c5.err
