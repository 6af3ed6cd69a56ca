#!/bin/bash
# usage: tools/gpu_prof_hbm.sh <tag> ; ncu full captures of the HBM-bound shapes: cfg5 n = 64 (bench.py)
# and cfg3 mode 0 (project(), k-tiled Omega), plus the cfg3 launch list
tag=${1:-hbm}
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:shgemm_sm100 -s 3 -c 1 \
   -o gpurun_out/${tag}_cfg5n64 python bench.py --config cfg5n64 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline \
   > gpurun_out/${tag}_ncu_a.txt 2>&1
echo "ncu_a exit $?" >> gpurun_out/${tag}_ncu_a.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:shgemm_sm100 -s 2 -c 1 \
   -o gpurun_out/${tag}_cfg3m0 python tools/proj_one.py > gpurun_out/${tag}_ncu_b.txt 2>&1
echo "ncu_b exit $?" >> gpurun_out/${tag}_ncu_b.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/${tag}_cfg3_launches.csv python tools/proj_one.py > gpurun_out/${tag}_ncu_c.txt 2>&1
echo "ncu_c exit $?" >> gpurun_out/${tag}_ncu_c.txt
