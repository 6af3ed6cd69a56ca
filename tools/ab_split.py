"""A/B of split-K / BN choices on the shapes where tiles < 2 waves (cfg2 projection, cfg3 modes)."""
import json
import sys

sys.path.insert(0, '.')
from tools.ab import run  # noqa: E402

allres = []
allres += run((16384, 16384, 272), [('auto', None), ('sk2', {'split_k': 2}), ('sk3', {'split_k': 3}),
                                    ('sk4', {'split_k': 4}), ('bn96_sk1', {'bn': 96}), ('bn96_sk2', {'bn': 96, 'split_k': 2})])
allres += run((1024, 1 << 20, 64), [('auto', None), ('sk37', {'split_k': 37}), ('sk36', {'split_k': 36}),
                                    ('sk74', {'split_k': 74})])
json.dump(allres, open('gpurun_out/ab_split.json', 'w'), indent=1)
