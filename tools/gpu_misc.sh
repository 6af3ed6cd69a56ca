#!/bin/bash
mkdir -p gpurun_out
# 1) 2-rank sharded bench on one GPU (gloo plumbing), cfg4 halves
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 \
    bench.py --gpus 2 --steps 3 --warmup 3 --no-e2e > gpurun_out/misc_bench2.json 2> gpurun_out/misc_bench2.err
echo "bench2 exit $?" >> gpurun_out/misc_bench2.err
# 2) compute-sanitizer on small shapes
for tool in memcheck racecheck synccheck; do
  timeout 600 compute-sanitizer --tool $tool --print-limit 20 python tools/hangdbg.py 0 300 700 160 > gpurun_out/misc_san_$tool.txt 2>&1
  echo "exit $?" >> gpurun_out/misc_san_$tool.txt
done
timeout 600 compute-sanitizer --tool memcheck --print-limit 20 python tools/hangdbg.py 0 600 1000 256 > gpurun_out/misc_san_memcheck_pair.txt 2>&1
echo "exit $?" >> gpurun_out/misc_san_memcheck_pair.txt
# 3) cfg3 mode-0 access pattern: TMA-only ablation vs full, and a cfg5-like 4-MB-stride control
python - > gpurun_out/misc_cfg3.txt 2>&1 <<'PY'
import sys, json, torch
sys.path.insert(0, '.')
from tools.ab import run
run((1024, 1 << 20, 64), [('full', None), ('tma_only', {'debug_flags': 7}), ('tma_only_nosplitk', {'debug_flags': 7, 'split_k': 9})], rounds=3)
run((8192, 1 << 17, 64), [('full', None), ('tma_only', {'debug_flags': 7})], rounds=3)
run((32768, 32768, 64), [('full', None), ('tma_only', {'debug_flags': 7})], rounds=3)
PY
