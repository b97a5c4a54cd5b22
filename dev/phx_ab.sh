#!/bin/bash
# philox fine sweep and config-4 run timing for the in-tree lib and dev/ab variants
for lib in "" $(ls dev/ab/libmmpr_*.so 2>/dev/null); do
  echo "== ${lib:-in-tree}"
  MMPR_LIB=$lib timeout 120 python dev/ncu_philox.py 2>&1 | tail -1
  MMPR_LIB=$lib NP_N=8 timeout 120 python dev/ncu_philox.py 2>&1 | tail -1
  MMPR_LIB=$lib timeout 120 python dev/phx_run_time.py 2>&1 | tail -1
done
