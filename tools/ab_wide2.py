"""Wide-tile timing (cfg2 projection, n = 288, TCEC line 3) with per-stage cycles and effective clock
(profiles/r02_wide2.jsonl): the round-2 wide schedule (part 1 promoted every second stage)."""
import json
import sys

sys.path.insert(0, '.')
from tools.ab import run  # noqa: E402

if __name__ == '__main__':
    allres = []
    for shape in [(16384, 16384, 272), (32768, 32768, 288), (1 << 21, 4096, 272)]:
        allres += run(shape, [('auto', None), ('single', {'pair': 2})], rounds=5, reps=10)
    with open('gpurun_out/r02_wide2.jsonl', 'w') as f:
        for r in allres:
            f.write(json.dumps(r) + '\n')
