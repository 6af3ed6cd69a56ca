"""A/B of the stream-K schedule (tune stream_k = 1) against whole tiles (stream_k = 2), interleaved on
the same inputs: median ms, cycles per stage and effective SM clock (profiles/r02_ab_streamk*.jsonl)."""
import json
import sys

sys.path.insert(0, '.')
from tools.ab import run  # noqa: E402

SHAPES = [(16384, 16384, 272), (32768, 32768, 256), (32768, 32768, 128), (8192, 16384, 256), (20000, 8192, 192)]

if __name__ == '__main__':
    shapes = [tuple(int(x) for x in a.split('x')) for a in sys.argv[2:]] or SHAPES
    out = sys.argv[1] if len(sys.argv) > 1 else 'gpurun_out/r02_ab_streamk.jsonl'
    allres = []
    for shape in shapes:
        allres += run(shape, [('tiles', {'stream_k': 2}), ('stream_k', {'stream_k': 1})], rounds=7, reps=10)
    with open(out, 'w') as f:
        for r in allres:
            f.write(json.dumps(r) + '\n')
