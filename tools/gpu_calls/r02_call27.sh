#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
bash tools/tg_prof_sweep.sh 16 48 18 50 > gpurun_out/tgsweep27.log 2>&1
