"""Run a script with the native library loaded from another path (A/B of build variants):
python tools/with_lib.py path/to/libcorridor_b200.so tools/prof_eizo14.py 2"""
import runpy, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2504_10783_b200 import _native as N

lib = N.load_library(sys.argv[1])
N._lib = lib
sys.argv = sys.argv[2:]
runpy.run_path(sys.argv[0], run_name="__main__")
