#!/bin/bash
# usage: tools/r02_gpu.sh <tag> [pytest args...]: GPU test suite (or a subset) then the default bench line
tag=${1:-r02}; shift
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv > gpurun_out/${tag}_smi.txt 2>&1
timeout 2400 python -m pytest ${@:-tests} -m gpu -q -rf -p no:cacheprovider > gpurun_out/${tag}_pytest.txt 2>&1
echo "pytest exit $?" >> gpurun_out/${tag}_pytest.txt
timeout 900 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
echo "bench exit $?" >> gpurun_out/${tag}_bench.err
