#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
for cfg in "0 256" "1 256" "3 256" "7 256" "7 32768" "0 32768"; do
  set -- $cfg
  echo "dbg=$1 chunk=$2: $(GANQ_HESSIAN_DBG=$1 GANQ_HESSIAN_CHUNK=$2 python tools/hess_iso.py 2>&1 | head -1)"
done > gpurun_out/hess10.log
