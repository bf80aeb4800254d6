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
    "tm3x4": ["SPC_TM_CTAS=3", "SPC_TM_NST=4"],
    "tm2x6": ["SPC_TM_CTAS=2", "SPC_TM_NST=6"],
    "tm5x2": ["SPC_TM_CTAS=5", "SPC_TM_NST=2"],
    "tmnomath": ["SPC_TM_NOMATH"],
    "tm3x4nm": ["SPC_TM_CTAS=3", "SPC_TM_NST=4", "SPC_TM_NOMATH"],
    "tm6x2": ["SPC_TM_CTAS=6", "SPC_TM_NST=2"],
    "evf": ["SPC_TM_EVICT_FIRST"],
    "ltnomath": ["SPC_LT_NOMATH"],
    "tmc2": ["SPC_TM_NCONS=2"],
    "tmc3": ["SPC_TM_NCONS=3"],
    "tmc2x6": ["SPC_TM_NCONS=2", "SPC_TM_CTAS=6", "SPC_TM_NST=2"],
    "tmc3x5": ["SPC_TM_NCONS=3", "SPC_TM_CTAS=5", "SPC_TM_NST=2"],
    "tmc2x5": ["SPC_TM_NCONS=2", "SPC_TM_CTAS=5", "SPC_TM_NST=2"],
    "ltb1": ["SPC_LT_BATCH=1"],
    "ltb2": ["SPC_LT_BATCH=2"],
    "ltnocvt": ["SPC_LT_EXP_NOCVT"],
    "sel1024": ["SPC_SEL_ST=1024"],
    "fixint": ["SPC_FIXPOINT_INT"],
    "vlsu": ["SPC_TM_VLSU=1"],
    "selearly": ["SPC_SEL_EARLY_LOADS"],
    "pf2": ["SPC_TM_PF=2"],
    "pf6": ["SPC_TM_PF=6"],
    "pf8": ["SPC_TM_PF=8"],
    "evn": ["SPC_TM_EVICT_NORMAL"],
    "ltnc4": ["SPC_LT_NC=4", "SPC_LT_CPR=1"],
}
for name in (sys.argv[1:] or VARIANTS):
    out = os.path.join(os.path.dirname(os.path.abspath(__file__)), f"libspc_{name}.so")
    build.build(out=out, defines=VARIANTS[name])
    print(out)
