#!/bin/bash
# usage: tools/r02_prof.sh <tag>: ncu launch list of the default bench (cfg4) + ncu --set full of the
# dominant kernel on cfg4, cfg5 n=1024 and cfg2's projection (profiles/r02_ncu_*); no bench numbers
tag=${1:-r02prof}
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 6 -c 8 --csv \
   --log-file gpurun_out/${tag}_launches_cfg4.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-extras \
   > gpurun_out/${tag}_ncu_launch_stdout.txt 2>&1
echo "ncu launches exit $?" >> gpurun_out/${tag}_ncu.err
for c in cfg4 cfg5n1024 cfg2proj; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:shgemm_sm100 -s 3 -c 1 \
   -o gpurun_out/${tag}_${c} python bench.py --config $c --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-extras \
   > gpurun_out/${tag}_ncu_full_${c}.txt 2>&1
echo "ncu full $c exit $?" >> gpurun_out/${tag}_ncu.err
done
