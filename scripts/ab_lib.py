"""A/B: time profile_c3-style runs against an alternative libhetreco_b200.so.
    python scripts/ab_lib.py <lib.so> <profile_c3 args...>"""
import os
import runpy
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1807_11830_b200 import hetreco as h  # noqa: E402

h.LIB_PATH = os.path.abspath(sys.argv[1])
sys.argv = ["profile_c3.py"] + sys.argv[2:]
runpy.run_path(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profile_c3.py"), run_name="__main__")
