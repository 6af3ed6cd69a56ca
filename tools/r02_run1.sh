#!/bin/bash
# round-2 first GPU check: bench (cfg4 + extras), ncu DRAM bytes of cfg5 n=1024, GPU tests
tag=${1:-r02a}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv > gpurun_out/${tag}_smi.txt 2>&1
timeout 900 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
echo "bench exit $?" >> gpurun_out/${tag}_bench.err
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second
for c in cfg5n1024 cfg4; do
timeout 600 ncu --metrics $M --clock-control none -k regex:shgemm_sm100 -c 2 --csv --log-file gpurun_out/${tag}_ncu_${c}.csv \
   python bench.py --config $c --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-extras > /dev/null 2>&1
echo "ncu $c exit $?" >> gpurun_out/${tag}_bench.err
done
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/${tag}_pytest.txt 2>&1
echo "pytest exit $?" >> gpurun_out/${tag}_pytest.txt
