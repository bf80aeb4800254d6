"""Run pytest with libspc replaced by a debug/variant build (tools only):
python tools/run_test_lib.py <lib.so> <pytest args...>"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_00722_b200 import spc  # noqa: E402

spc._lib = spc.load_library(sys.argv[1])
import pytest  # noqa: E402

sys.exit(pytest.main(sys.argv[2:]))
