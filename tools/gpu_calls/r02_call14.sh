#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/gpu_suite14.log 2>&1
python tools/sanitize_case.py > gpurun_out/san_plain14.log 2>&1 && \
timeout 1500 compute-sanitizer --tool racecheck --racecheck-report all python tools/sanitize_case.py > gpurun_out/racecheck14.log 2>&1
