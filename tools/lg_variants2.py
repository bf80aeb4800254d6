"""Build LOGITS variants (tools/libspc_<name>.so) with -D flags (tools only; run on CPU)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_00722_b200 import build  # noqa: E402

VARIANTS = {
    "nomath": ["SPC_LT_NOMATH"],
    "nc4": ["SPC_LT_NC=4", "SPC_LT_CPR=1"],
    "b1": ["SPC_LT_BATCH=1"],
    "b4": ["SPC_LT_BATCH=4"],
    "scl16": ["SPC_SEL_SCL=16"],
    "nreg80": ["SPC_SEL_NREG=80"],
}
for name in (sys.argv[1:] or VARIANTS):
    out = os.path.join(os.path.dirname(os.path.abspath(__file__)), f"libspc_{name}.so")
    build.build(out=out, defines=VARIANTS[name])
    print(out)
