#!/bin/bash
# final verification of the round-2 code: GPU suite, smoke, the default bench line
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/t55.log 2>&1
timeout 300 python -c "import __graft_entry__ as e; e.smoke(); print('smoke ok')" > gpurun_out/smoke55.log 2>&1
timeout 600 python bench.py > gpurun_out/bench55.json 2> gpurun_out/bench55.err
