"""A/B: row-major A staging with 128-B row visits (a_box 1) vs 256-B row visits (a_box 2)."""
import sys, json
sys.path.insert(0, '.'); sys.path.insert(0, 'tools')
from ab import run
allres = []
for shape in [(1024, 1 << 20, 64), (4096, 1 << 18, 64), (32768, 32768, 64), (32768, 32768, 128), (1 << 20, 4096, 256),
              (32768, 32768, 1024), (16384, 16384, 16)]:
    allres += run(shape, [('abox1', {'a_box': 1}), ('abox2', {'a_box': 2})], rounds=5, reps=3)
json.dump(allres, open('gpurun_out/ab_abox.json', 'w'), indent=1)
