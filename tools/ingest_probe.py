"""Instance load to device: file -> host arrays -> handle vs device ingest (pcb_create_from_file)."""
import os
import sys
import time
sys.path.insert(0, '/root/repo')
import numpy as np
from paracut_b200 import _native, io as pio
from paracut_b200.instances import make_instance

wl = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
g = make_instance(wl, seed=0)
path = "/tmp/%s.pcut" % wl
pio.write_grid(g, path)
del g
print("file %.0f MB" % (os.path.getsize(path) / 1e6))
for rep in range(3):
    os.system("sync")
    t0 = time.perf_counter()
    h = pio.read_grid(path)
    t1 = time.perf_counter()
    S = _native.GridSolver(h, precision="f32")
    S.synchronize()
    t2 = time.perf_counter()
    S.close(); del S, h
    t3 = time.perf_counter()
    S = _native.GridSolver(pio.open_grid(path), precision="f32")
    S.synchronize()
    t4 = time.perf_counter()
    S.close(); del S
    print("read_grid %.1f ms + create %.1f ms = %.1f ms | device ingest %.1f ms"
          % ((t1 - t0) * 1e3, (t2 - t1) * 1e3, (t2 - t0) * 1e3, (t4 - t3) * 1e3))
