"""Write the generated specialised-check source of the 7- or 14-DOF model (EZ_JIT_DUMP): python tools/dump_jit.py 7|14 [path]."""
import os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
os.environ["EZ_JIT_DUMP"] = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out/jit_franka7.cu"
from paper_2504_10783_b200 import fixtures as fx
w = {"7": fx.franka7_world, "14": fx.bimanual14_world}[sys.argv[1] if len(sys.argv) > 1 else "7"]()
w.checker(specialize=False).native.specialize(1)
