"""Dev probe: load cubins with the driver API and print the launch limits
(max threads per block, registers, static/local memory) of their qk_jit kernel."""
import ctypes
import sys

cu = ctypes.CDLL("libcuda.so.1")
cu.cuInit(0)
dev = ctypes.c_int()
cu.cuDeviceGet(ctypes.byref(dev), 0)
ctx = ctypes.c_void_p()
cu.cuDevicePrimaryCtxRetain(ctypes.byref(ctx), dev)
cu.cuCtxSetCurrent(ctx)
ATTR = {"max_threads": 0, "shared_static": 1, "const": 2, "local": 3, "regs": 4, "max_dyn_smem": 8}
for path in sys.argv[1:]:
    data = open(path, "rb").read()
    mod = ctypes.c_void_p()
    rc = cu.cuModuleLoadData(ctypes.byref(mod), data)
    fn = ctypes.c_void_p()
    rc2 = cu.cuModuleGetFunction(ctypes.byref(fn), mod, b"qk_jit")
    vals = {}
    for k, a in ATTR.items():
        v = ctypes.c_int()
        cu.cuFuncGetAttribute(ctypes.byref(v), a, fn)
        vals[k] = v.value
    print(path.split("/")[-1][:20], rc, rc2, vals)
