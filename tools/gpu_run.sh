#!/bin/bash
# usage: tools/gpu_run.sh <tag> ; runs gpu tests + quick perf, writes into gpurun_out/
tag=${1:-run}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${tag}_smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -rf --timeout=600 -p no:cacheprovider > gpurun_out/${tag}_pytest.txt 2>&1
echo "pytest exit $?" >> gpurun_out/${tag}_pytest.txt
timeout 600 python tools/quick_perf.py > gpurun_out/${tag}_perf.txt 2>&1
echo "perf exit $?" >> gpurun_out/${tag}_perf.txt
