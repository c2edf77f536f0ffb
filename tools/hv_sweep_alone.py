import ctypes, os, sys
sys.path.insert(0, '/root/repo')
os.environ['ML_LIB'] = 'build_dbg/libml_hv.so'
import mlgen, paper_1607_00315_b200 as ml
ds = mlgen.make(5)
ctx = ml.Context(ds)
ctx.ml_set_engine(16)
L = ml.load()
L.ml_debug_hv_sweep.restype = ctypes.c_double
L.ml_debug_hv_sweep.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int]
print("sweep alone ms NV=1", L.ml_debug_hv_sweep(ctx.h, 5, 1), "NV=2", L.ml_debug_hv_sweep(ctx.h, 5, 2), ctx.ml_heavy_info())
