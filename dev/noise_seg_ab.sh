#!/bin/bash
# A/B of the segmented warp fill (launch bounds, segment counts) against the unsegmented 8-word kernel
O=gpurun_out/${TAG:-noise_seg}
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_noise.py -x -q > $O/pytest_noise.log 2>&1; echo "rc=$?" >> $O/pytest_noise.log
{
for segs in -1 0 1 4 16; do echo "== default lib MMPR_NOISE_SEGS=$segs"; MMPR_NOISE_SEGS=$segs timeout 300 python dev/noise_ab.py; done
for v in ns24 ns20 ns16; do for segs in 0 1 8; do echo "== $v MMPR_NOISE_SEGS=$segs"; MMPR_LIB=dev/ab/libmmpr_$v.so MMPR_NOISE_SEGS=$segs timeout 300 python dev/noise_ab.py; done; done
} > $O/ab.log 2>&1
tail -5 $O/pytest_noise.log; cat $O/ab.log
