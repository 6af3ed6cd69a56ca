"""Per-role wait cycles and ablations for the wide-N tile (BN 272) vs BN 256 at the tall shape."""
import sys

sys.path.insert(0, ".")
from tools.diag import run  # noqa: E402

run("wide", [(1 << 21, 4096, 272)], flags_list=(0, 1, 2, 4, 8))
run("n256", [(1 << 21, 4096, 256)], flags_list=(0, 1, 4))
