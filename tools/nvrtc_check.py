"""Compile a generated specialised-check source (EZ_JIT_DUMP) with NVRTC on the CPU, as ez_jit.cu does."""
import ctypes as C, sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2504_10783_b200.build import JIT_HEADERS

nv = C.CDLL("/usr/local/cuda/lib64/libnvrtc.so.12")
src = Path(sys.argv[1]).read_text()
names = [n.encode() for n, _ in JIT_HEADERS]
texts = [p.read_text().encode() for _, p in JIT_HEADERS]
prog = C.c_void_p()
arr = lambda xs: (C.c_char_p * len(xs))(*xs)
assert nv.nvrtcCreateProgram(C.byref(prog), src.encode(), b"jit.cu", len(names), arr(texts), arr(names)) == 0
opts = [b"--gpu-architecture=sm_100a", b"--std=c++17", b"-lineinfo"] + [a.encode() for a in sys.argv[2:]]
r = nv.nvrtcCompileProgram(prog, len(opts), arr(opts))
n = C.c_size_t()
nv.nvrtcGetProgramLogSize(prog, C.byref(n))
log = C.create_string_buffer(n.value)
nv.nvrtcGetProgramLog(prog, log)
print("result", r)
print(log.value.decode()[:5000])
if r == 0:
    nv.nvrtcGetCUBINSize(prog, C.byref(n))
    buf = C.create_string_buffer(n.value)
    nv.nvrtcGetCUBIN(prog, buf)
    Path("/tmp/jit.cubin").write_bytes(buf.raw)
    print("cubin bytes", n.value, "-> /tmp/jit.cubin")
