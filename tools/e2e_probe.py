"""Time pk_run_host (host buffers, PCIe inside) for the headline matmul (development aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1801_04348_b200 import _lib
if len(sys.argv) > 1:
    _lib.LIB_PATH = os.path.abspath(sys.argv[1])
import time, torch, numpy as np
from paper_1801_04348_b200 import binding, cases, programs
n=8192
kind=programs.original("matmul"); P={"n":n,"B0":128,"ub1":8,"s":int(sys.argv[2]) if len(sys.argv)>2 else 8}
sel=cases.select(kind,P,"live")
L=binding.make_launch(kind,P,sel.applied,_lib.DTYPE_F32)
hs=[torch.rand(n*n).pin_memory() for _ in range(3)]
for i in range(2): _lib.run_host(L,[h.data_ptr() for h in hs],0)
t=time.time(); R=5
for i in range(R): _lib.run_host(L,[h.data_ptr() for h in hs],0)
dt=(time.time()-t)/R
print(sys.argv[1:], "e2e run_host n=8192: %.2f ms  %.1f GFLOP/s"%(dt*1e3, 2*n**3/dt/1e9))
