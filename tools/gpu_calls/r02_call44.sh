#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 600 bash tools/ss_prof.sh 16 c3 > gpurun_out/ssprof44_c3.log 2>&1
