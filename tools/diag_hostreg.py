"""Cost of registering (cudaHostRegister) a pageable 28 MB row array instead of copying it into pinned stages (DESIGN: slower than copying)."""
import time, numpy as np, torch
cr = torch.cuda.cudart()
torch.cuda.init()
for trial in range(3):
    a = np.random.default_rng(0).uniform(size=(1 << 20, 7)).astype(np.float32)
    t0 = time.perf_counter()
    r = cr.cudaHostRegister(a.ctypes.data, a.nbytes, 0)
    t1 = time.perf_counter()
    cr.cudaHostUnregister(a.ctypes.data)
    t2 = time.perf_counter()
    print(f"register {1e3*(t1-t0):.3f} ms (rc {r}) unregister {1e3*(t2-t1):.3f} ms")
    import ctypes
    libc = ctypes.CDLL("libc.so.6")
    b = np.empty((1 << 20, 7), np.float32)
    libc.madvise(ctypes.c_void_p(b.ctypes.data & ~((1 << 21) - 1)), ctypes.c_size_t(b.nbytes + (1 << 21)), 14)  # MADV_HUGEPAGE
    b[:] = a
    t0 = time.perf_counter()
    r = cr.cudaHostRegister(b.ctypes.data, b.nbytes, 0)
    t1 = time.perf_counter()
    cr.cudaHostUnregister(b.ctypes.data)
    print(f"  THP-advised: register {1e3*(t1-t0):.3f} ms")
print(open("/sys/kernel/mm/transparent_hugepage/enabled").read())
