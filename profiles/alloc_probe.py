"""How long does it take to obtain 64 GiB of device memory (cudaMalloc vs
cudaMallocAsync pool growth, first and second time), first touch (memset) included?  Explains the first-call
cost of preconditioned_components at c4/c5 (X~ is a fresh 64 GiB buffer)."""
import ctypes, time, json
import torch
torch.cuda.init()
rt = ctypes.CDLL("libcudart.so.12") if False else None
import glob, os
cands = glob.glob(os.path.join(os.path.dirname(torch.__file__), "lib", "libcudart*.so*")) + \
    glob.glob("/usr/local/cuda/lib64/libcudart.so*")
rt = ctypes.CDLL(cands[0])
GB = 1 << 30
res = {}
def t_malloc(nbytes):
    p = ctypes.c_void_p()
    rt.cudaDeviceSynchronize(); t0 = time.perf_counter()
    rc = rt.cudaMalloc(ctypes.byref(p), ctypes.c_size_t(nbytes)); rt.cudaMemset(p, 0, ctypes.c_size_t(nbytes)); rt.cudaDeviceSynchronize()
    t1 = time.perf_counter(); rt.cudaFree(p); rt.cudaDeviceSynchronize(); t2 = time.perf_counter()
    return rc, t1 - t0, t2 - t1
def t_malloc_async(nbytes):
    p = ctypes.c_void_p()
    rt.cudaDeviceSynchronize(); t0 = time.perf_counter()
    rc = rt.cudaMallocAsync(ctypes.byref(p), ctypes.c_size_t(nbytes), None); rt.cudaMemset(p, 0, ctypes.c_size_t(nbytes)); rt.cudaDeviceSynchronize()
    t1 = time.perf_counter(); rt.cudaFreeAsync(p, None); rt.cudaDeviceSynchronize(); t2 = time.perf_counter()
    return rc, t1 - t0, t2 - t1
for g in (1, 8, 64):
    res[f"cudaMalloc_{g}G"] = t_malloc(g * GB)
    res[f"cudaMalloc_{g}G_again"] = t_malloc(g * GB)
# default pool, release threshold max (as the library sets it)
pool = ctypes.c_void_p()
rt.cudaDeviceGetDefaultMemPool(ctypes.byref(pool), 0)
thr = ctypes.c_uint64(2**64 - 1)
rt.cudaMemPoolSetAttribute(pool, 4, ctypes.byref(thr))  # cudaMemPoolAttrReleaseThreshold = 4
for g in (1, 8, 64):
    res[f"cudaMallocAsync_{g}G"] = t_malloc_async(g * GB)
    res[f"cudaMallocAsync_{g}G_again"] = t_malloc_async(g * GB)
print(json.dumps({k: [v[0], round(v[1], 4), round(v[2], 4)] for k, v in res.items()}))
