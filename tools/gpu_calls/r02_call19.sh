#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -s -k "sstep_teacher" > gpurun_out/t19.log 2>&1
GANQ_SSTEP_DBG=16 true
