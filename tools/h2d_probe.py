import time, torch, numpy as np, os
n = 535*1024*1024//8
a = np.random.default_rng(0).normal(size=n)
d = torch.empty(n, dtype=torch.float64, device='cuda')
for rep in range(3):
    t=time.perf_counter(); d.copy_(torch.from_numpy(a)); torch.cuda.synchronize(); dt=time.perf_counter()-t
    print("pageable H2D %.1f GB/s" % (a.nbytes/dt/1e9))
p = torch.empty(n, dtype=torch.float64).pin_memory()
for rep in range(3):
    t=time.perf_counter(); d.copy_(p, non_blocking=True); torch.cuda.synchronize(); dt=time.perf_counter()-t
    print("pinned H2D %.1f GB/s" % (a.nbytes/dt/1e9))
for rep in range(3):
    t=time.perf_counter(); p.copy_(d, non_blocking=True); torch.cuda.synchronize(); dt=time.perf_counter()-t
    print("pinned D2H %.1f GB/s" % (a.nbytes/dt/1e9))
b = np.empty_like(a)
for rep in range(3):
    t=time.perf_counter(); torch.from_numpy(b).copy_(d); torch.cuda.synchronize(); dt=time.perf_counter()-t
    print("pageable D2H %.1f GB/s" % (a.nbytes/dt/1e9))
for rep in range(2):
    t=time.perf_counter(); np.copyto(p.numpy(), a); dt=time.perf_counter()-t
    print("host memcpy 1 thread %.1f GB/s" % (a.nbytes/dt/1e9))
import ctypes
t=time.perf_counter(); r=torch.cuda.cudart().cudaHostRegister(a.ctypes.data, a.nbytes, 0); dt=time.perf_counter()-t
print("hostRegister %.1f ms rc %s" % (dt*1e3, r))
for rep in range(2):
    t=time.perf_counter(); d.copy_(torch.from_numpy(a), non_blocking=True); torch.cuda.synchronize(); dt=time.perf_counter()-t
    print("registered H2D %.1f GB/s" % (a.nbytes/dt/1e9))
print("cpus", os.cpu_count(), len(os.sched_getaffinity(0)))
