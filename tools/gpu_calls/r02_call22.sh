#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/gpu_suite22.log 2>&1
python bench.py --steps 20 --warmup 5 > gpurun_out/bench22.json 2> gpurun_out/bench22.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench22_ref.json 2> gpurun_out/bench22_ref.err
python -c "import __graft_entry__ as e; e.smoke(); print('smoke ok')" > gpurun_out/smoke22.log 2>&1
python tools/scale_projection.py --config c3 > gpurun_out/scale22_c3.jsonl 2> gpurun_out/scale22_c3.err
python tools/configs_run.py all > gpurun_out/configs22.jsonl 2> gpurun_out/configs22.err
