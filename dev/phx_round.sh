#!/bin/bash
# Philox-mode check: parity tests, fine-sweep timing, the other-config timings
O=gpurun_out/${TAG:-phx}
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_philox.py -x -q > $O/pytest_philox.log 2>&1; echo "rc=$?" >> $O/pytest_philox.log
timeout 300 python dev/ncu_philox.py > $O/philox_sweep.log 2>&1
NP_N=8 timeout 300 python dev/ncu_philox.py >> $O/philox_sweep.log 2>&1
timeout 600 python -c "import json, torch, bench; import paper_2310_11365_b200 as mm; print(json.dumps(bench.other_configs(mm, torch), indent=1))" > $O/configs.json 2> $O/configs.err
${EXTRA:-true}
