#!/bin/bash
# ncu --set full of the dominant kernel on the HBM-bound cfg5 points (n = 64, 128; stream-K plans)
tag=${1:-r02hbm}
mkdir -p gpurun_out
for c in cfg5n64 cfg5n128; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:shgemm_sm100 -s 3 -c 1 \
   -o gpurun_out/${tag}_${c} python bench.py --config $c --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-extras \
   > gpurun_out/${tag}_ncu_full_${c}.txt 2>&1
echo "ncu full $c exit $?" >> gpurun_out/${tag}_ncu.err
done
