"""Per-role waits and ablations on the HBM-bound shapes (cfg5 n = 16 / 64 / 128, cfg3 mode 0)."""
import sys

sys.path.insert(0, ".")
from tools.diag import run  # noqa: E402

run("hbm", [(32768, 32768, 16), (32768, 32768, 64), (32768, 32768, 128), (1024, 1 << 20, 64)],
    flags_list=(0, 1, 2, 4, 8, 15))
