"""A/B of Omega multicast (tune omega_mcast = 1 / 2 / 4 pairs per cluster) on the pair shapes."""
import json
import sys

sys.path.insert(0, '.')
from tools.ab import run  # noqa: E402

allres = []
V = [('mc1', {'omega_mcast': 1}), ('mc2', {'omega_mcast': 2}), ('mc3', {'omega_mcast': 3}), ('mc4', {'omega_mcast': 4})]
for shape in [(1 << 22, 4096, 256), (32768, 32768, 256), (32768, 32768, 1024), (32768, 32768, 128), (16384, 16384, 272)]:
    allres += run(shape, V)
json.dump(allres, open('gpurun_out/ab_mcast.json', 'w'), indent=1)
