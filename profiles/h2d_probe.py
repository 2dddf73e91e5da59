import sys, time, ctypes, numpy as np
sys.path.insert(0, ".")
import paper_2008_11476_b200 as gvx
c, g = gvx._load()
c.gvxb_host_register.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
dev = gvx.Device(0)
n = 3840 * 2160
a = np.ones(n, np.uint8)
print("register", c.gvxb_host_register(a.ctypes.data, n), file=sys.stderr)
d = dev.alloc(n)
for k in range(4):
    dev.sync(); t = time.perf_counter()
    c.gvxb_upload_2d(dev.h, ctypes.c_void_p(d), 3840, a.ctypes.data, 3840, 3840, 2160)
    dev.sync(); dt = time.perf_counter() - t
    print("gvxb_upload_2d registered GB/s", n / dt / 1e9, file=sys.stderr)
# legacy stream
c.gvxb_ctx_set_stream(dev.h, None)
for k in range(3):
    dev.sync(); t = time.perf_counter()
    c.gvxb_upload_2d(dev.h, ctypes.c_void_p(d), 3840, a.ctypes.data, 3840, 3840, 2160)
    dev.sync(); dt = time.perf_counter() - t
    print("legacy stream GB/s", n / dt / 1e9, file=sys.stderr)
# freshly written (cache-resident, dirty) source
for k in range(3):
    a[:] = k
    dev.sync(); t = time.perf_counter()
    c.gvxb_upload_2d(dev.h, ctypes.c_void_p(d), 3840, a.ctypes.data, 3840, 3840, 2160)
    dev.sync(); dt = time.perf_counter() - t
    print("just-written source GB/s", n / dt / 1e9, file=sys.stderr)
import platform, os
print(platform.machine(), os.cpu_count(), open("/proc/cpuinfo").read().split("model name")[1].split("\n")[0], file=sys.stderr)
# heap (brk) memory from malloc, registered
libc = ctypes.CDLL("libc.so.6")
libc.malloc.restype = ctypes.c_void_p
libc.malloc.argtypes = [ctypes.c_size_t]
libc.mallopt.argtypes = [ctypes.c_int, ctypes.c_int]
for label, thresh in (("mmap'ed malloc", None), ("brk heap malloc", 64 << 20)):
    if thresh:
        libc.mallopt(-3, thresh)  # M_MMAP_THRESHOLD
    p = libc.malloc(n)
    ctypes.memset(p, 1, n)
    print(label, hex(p), "register", c.gvxb_host_register(ctypes.c_void_p(p), n), file=sys.stderr)
    for k in range(3):
        dev.sync(); t = time.perf_counter()
        c.gvxb_upload_2d(dev.h, ctypes.c_void_p(d), 3840, ctypes.c_void_p(p), 3840, 3840, 2160)
        dev.sync(); dt = time.perf_counter() - t
        print(label, "H2D GB/s", n / dt / 1e9, file=sys.stderr)
    for k in range(2):
        dev.sync(); t = time.perf_counter()
        c.gvxb_download_2d(dev.h, ctypes.c_void_p(p), 3840, ctypes.c_void_p(d), 3840, 3840, 2160)
        dev.sync(); dt = time.perf_counter() - t
        print(label, "D2H GB/s", n / dt / 1e9, file=sys.stderr)
