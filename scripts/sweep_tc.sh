#!/bin/bash
# Development sweep of tcgen05 tile configs (CBB_TC_CFG) x epilogue modes (CBB_TC_EPI_MODE).
mkdir -p gpurun_out
for cfg in ${CFGS:-0 1 2 3 4 5}; do
  for m in ${MODES:-2 0}; do
    echo "cfg=$cfg mode=$m $(CBB_TC_CFG=$cfg CBB_TC_EPI_MODE=$m timeout 120 python scripts/probe_cfg1.py ${N:-1048576} ${D:-131072} tcgen05 2>&1 | grep it3)"
  done
done
