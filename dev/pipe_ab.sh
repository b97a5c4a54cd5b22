#!/bin/bash
# A/B of the config-4 run: in-tree library vs the builds in dev/ab/, alternating.
for i in 1 2; do
  python dev/pipe_sweep.py MMPR_PIPELINE_CLUSTERS=14 2>&1 | sed 's/^/new  /'
  for lib in dev/ab/*.so; do
    MMPR_LIB=$PWD/$lib python dev/pipe_sweep.py MMPR_PIPELINE_CLUSTERS=14 2>&1 | sed "s#^#$(basename $lib) #"
  done
done
