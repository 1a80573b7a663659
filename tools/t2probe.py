import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
from paper_1801_04348_b200 import _lib, binding, cases, programs
P={"T":50,"N":16386,"s":16,"B0":8,"B1":32}
kind=programs.original("jacobi2d"); sel=cases.select(kind,P,"live")
a=torch.randint(-(1<<20),1<<20,(2*16386*16386,),dtype=torch.int32,device="cuda")
st=torch.cuda.current_stream().cuda_stream
for h in (0,3,5,7,9,11):
    L=binding.make_launch(kind,P,sel.applied,_lib.DTYPE_I32,extra_flags=_lib.FLAG_TEMPORAL if h else 0)
    if h: L.tblock=h
    _lib.launch(L,[a.data_ptr()],st); torch.cuda.synchronize()
    e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
    e0.record(); _lib.launch(L,[a.data_ptr()],st); e1.record(); torch.cuda.synchronize()
    ms=e0.elapsed_time(e1); print("h=%d %.2f ms %.1f GB/s-equiv"%(h,ms,50*8*16384**2/ms/1e6), flush=True)
