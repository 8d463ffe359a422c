"""C2 step timing with an alternative library build (argv[1]: path to libkerntune_b200.so)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2102_04199_b200 import _lib  # noqa: E402

if len(sys.argv) > 1:
    _lib._lib = _lib.load(sys.argv[1])
sys.argv = sys.argv[:1]
import runpy  # noqa: E402

runpy.run_path(os.path.join(os.path.dirname(os.path.abspath(__file__)), "pretrain_quick.py"), run_name="__main__")
