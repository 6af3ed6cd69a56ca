#!/bin/bash
# usage: tools/r02_final.sh <tag>: HEAD check — GPU suite, smoke, default bench line, ncu launch list of
# the bench, project() fuzz (in-kernel Omega drawn)
tag=${1:-r02final}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv > gpurun_out/${tag}_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${tag}_pytest.txt 2>&1
echo "pytest exit $?" >> gpurun_out/${tag}_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.txt 2>&1
echo "smoke exit $?" >> gpurun_out/${tag}_smoke.txt
timeout 900 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
echo "bench exit $?" >> gpurun_out/${tag}_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 6 -c 8 --csv \
   --log-file gpurun_out/${tag}_launches_cfg4.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-extras \
   > gpurun_out/${tag}_ncu_launch_stdout.txt 2>&1
echo "ncu exit $?" >> gpurun_out/${tag}_bench.err
timeout 600 python tools/fuzz_project_large.py 0 120 > gpurun_out/${tag}_fuzz_project_large.txt 2>&1
echo "fuzz exit $?" >> gpurun_out/${tag}_fuzz_project_large.txt
