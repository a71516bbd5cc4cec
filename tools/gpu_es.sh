#!/bin/bash
# ES breakdown: tests, timings, launch list, ncu captures of the sort pass / partial / gen kernels
mkdir -p gpurun_out
python -m pytest tests/test_es_device.py tests/test_dist_gpu.py -m gpu -x -q 2>&1 | tail -3
for T in 0 5 12 20; do TASK=$T python tools/es_probe.py; done
GENS=3 REPS=1 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/es_launches.csv python tools/es_probe.py > /dev/null 2>&1
if [ -n "$FULL" ]; then
  GENS=3 REPS=0 ncu --set full --clock-control none --import-source on -k regex:"rs_pass_kernel|es_partial_kernel|es_gen_kernel" -s 4 -c 4 -f -o gpurun_out/es_full python tools/es_probe.py > gpurun_out/es_full.log 2>&1
fi
