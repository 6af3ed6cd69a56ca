#!/bin/bash
# usage: tools/gpu_prof.sh <tag> ; bench + ncu launch list + ncu full capture of the shgemm kernel
tag=${1:-prof}
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
echo "bench exit $?" >> gpurun_out/${tag}_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 6 -c 8 --csv \
   --log-file gpurun_out/${tag}_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline \
   > gpurun_out/${tag}_ncu_launch_stdout.txt 2>&1
echo "ncu1 exit $?" >> gpurun_out/${tag}_bench.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:shgemm_sm100 -s 3 -c 1 \
   -o gpurun_out/${tag}_cfg4 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline \
   > gpurun_out/${tag}_ncu_full_stdout.txt 2>&1
echo "ncu2 exit $?" >> gpurun_out/${tag}_bench.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:shgemm_sm100 -s 3 -c 1 \
   -o gpurun_out/${tag}_cfg5n1024 python bench.py --config cfg5n1024 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline \
   > gpurun_out/${tag}_ncu_full2_stdout.txt 2>&1
echo "ncu3 exit $?" >> gpurun_out/${tag}_bench.err
