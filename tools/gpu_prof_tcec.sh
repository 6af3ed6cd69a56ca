#!/bin/bash
# usage: tools/gpu_prof_tcec.sh <tag> ; ncu launch list + one full capture of the TCEC-SGEMM mainloop
# (RSVD line 3 at cfg2: B^T = A^T Q, 16384 x 16384 MN-major A, n = 272)
tag=${1:-tcec}
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 12 --csv \
   --log-file gpurun_out/${tag}_launches.csv python tools/tcec_one.py > gpurun_out/${tag}_ncu1.txt 2>&1
echo "ncu1 exit $?" >> gpurun_out/${tag}_ncu1.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:shgemm_sm100 -s 2 -c 1 \
   -o gpurun_out/${tag}_full python tools/tcec_one.py > gpurun_out/${tag}_ncu2.txt 2>&1
echo "ncu2 exit $?" >> gpurun_out/${tag}_ncu2.txt
