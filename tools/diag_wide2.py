import sys, json
sys.path.insert(0, '.')
from tools.diag import run
res = run('w', [(16384, 16384, 272), (1 << 20, 4096, 256)], flags_list=(0, 1, 2, 4, 8))
json.dump(res, open('gpurun_out/r02_diag_wide2.json', 'w'), indent=1)
