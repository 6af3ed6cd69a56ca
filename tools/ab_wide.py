"""A/B: wide N tiles (BN 272/288, one A pass) vs two narrower tiles for 256 < n <= 288 and n = 544."""
import json
import sys

sys.path.insert(0, '.')
from tools.ab import run  # noqa: E402

allres = []
allres += run((16384, 16384, 272), [('wide272', None), ('bn144', {'bn': 144})])
allres += run((32768, 32768, 288), [('wide288', None), ('bn144', {'bn': 144})])
allres += run((32768, 32768, 544), [('wide272x2', None), ('bn192x3', {'bn': 192})])
allres += run((1 << 21, 4096, 272), [('wide272', None), ('bn144', {'bn': 144})])
json.dump(allres, open('gpurun_out/ab_wide.json', 'w'), indent=1)
