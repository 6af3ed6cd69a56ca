"""Per-role wait cycles and ablations for SHGEMM-TF32 vs SHGEMM-FP16 (tools/diag.py run())."""
import json, sys
sys.path.insert(0, '.'); sys.path.insert(0, 'tools')
from diag import run
shapes = [(1 << 20, 4096, 256), (32768, 32768, 64), (32768, 32768, 128), (32768, 32768, 16)]
flags = tuple(int(x) for x in sys.argv[1].split(',')) if len(sys.argv) > 1 else (0,)
res = run("fp16", shapes, flags_list=(0,))
res += run("tf32", shapes, flags_list=flags, extra_tune={"tc": 1})
json.dump(res, open("gpurun_out/diag_tf32.json", "w"), indent=1)
