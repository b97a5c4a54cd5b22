#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over small shapes of the
# hand-written protocols: the iteration pipeline (one rank; several ranks
# emulated in one launch, epoch-tagged flags, system-scope paths), the
# cluster fine sweep (mbarrier + st.async DSMEM exchange), the grid sweep
# (team counters through L2), the one-pass region restriction and the noise
# generator.  Each case is an existing GPU parity test, so a run also checks
# the results.  Output: gpurun_out/${TAG:-san}/<tool>_<case>.log + summary.txt
O=gpurun_out/${TAG:-san}
mkdir -p $O
CS=/usr/local/cuda/bin/compute-sanitizer
declare -A CASES=(
  [pipeline1]="tests/test_gpu_pipeline.py::test_pipeline_equals_per_iteration_kernels_ou[3-1-10-100000]"
  [pipeline_ranks]="tests/test_gpu_pipeline.py::test_multi_rank_pipeline_system_scope"
  [fine_cluster]="tests/test_gpu_fine.py::test_injected_mode_bitwise_ou[100000]"
  [fine_grid]="tests/test_gpu_fine.py::test_grid_variant_bitwise_ou[1048576-32-1-2]"
  [regions]="tests/test_gpu_regions.py::test_match_restrict_regions_equals_separate_passes[5000-0]"
  [noise]="tests/test_gpu_noise.py::test_slice_noise_matches_numpy[100000]"
  [philox_fine]="tests/test_gpu_philox.py::test_propagate_fine_counter_equals_oracle[ou-100000]"
  [philox_run]="tests/test_gpu_philox.py::test_run_philox_equals_oracle_with_counter_noise[True]"
)
: > $O/summary.txt
for tool in ${TOOLS:-memcheck racecheck synccheck}; do
  for c in ${!CASES[@]}; do
    log=$O/${tool}_${c}.log
    timeout ${CASE_TIMEOUT:-600} $CS --tool $tool --target-processes all --print-limit 20 \
      python -m pytest -q -p no:cacheprovider "${CASES[$c]}" > $log 2>&1
    rc=$?
    echo "$tool $c rc=$rc $(grep -h 'ERROR SUMMARY\|RACECHECK SUMMARY\|passed\|failed' $log | tr '\n' ' ')" >> $O/summary.txt
  done
done
cat $O/summary.txt
