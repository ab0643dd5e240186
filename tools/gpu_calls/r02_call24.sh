#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
bash tools/tg_prof_sweep.sh > gpurun_out/tgsweep24.log 2>&1
