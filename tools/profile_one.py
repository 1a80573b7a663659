"""Launch one family's case-selected kernel a few times (for ncu captures).

python tools/profile_one.py FAMILY '{"N": ..., ...}' [launches] [--generic] [--tf32x3] [--f32]
"""

import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1801_04348_b200 import _lib, binding, cases, programs  # noqa: E402
from paper_1801_04348_b200 import machine as machine_mod  # noqa: E402


def main():
    fam = sys.argv[1]
    params = json.loads(sys.argv[2])
    launches = int(sys.argv[3]) if len(sys.argv) > 3 and sys.argv[3].isdigit() else 3
    generic = "--generic" in sys.argv
    extra = _lib.FLAG_TF32X3 if "--tf32x3" in sys.argv else 0
    temporal = [int(a.split("=")[1]) for a in sys.argv if a.startswith("--temporal=")]
    if temporal:
        extra |= _lib.FLAG_TEMPORAL
    kind = programs.original(fam)
    mv = machine_mod.live()
    sel = cases.select(kind, params, mv)
    dtype = _lib.DTYPE_F32 if fam == "matmul" or "--f32" in sys.argv else _lib.DTYPE_I32
    if "--f64" in sys.argv:
        dtype = _lib.DTYPE_F64
        mv = machine_mod.live(elem_bytes=8)
        sel = cases.select(kind, params, mv)
    L = binding.make_launch(kind, params, sel.applied, dtype, generic=generic, extra_flags=extra)
    if temporal:
        L.tblock = temporal[0]
    shapes = programs.array_shapes(kind, params)
    bufs = []
    for a in programs.FAMILIES[fam].arrays:
        n = 1
        for d in shapes[a.name]:
            n *= d
        if dtype == _lib.DTYPE_F32:
            bufs.append(torch.rand(n, device="cuda") - 0.5)
        elif dtype == _lib.DTYPE_F64:
            bufs.append(torch.rand(n, device="cuda", dtype=torch.float64) - 0.5)
        else:
            bufs.append(torch.randint(-1000, 1000, (n,), dtype=torch.int32, device="cuda"))
    st = torch.cuda.current_stream().cuda_stream
    for _ in range(launches):
        _lib.launch(L, [b.data_ptr() for b in bufs], st)
    torch.cuda.synchronize()
    print(fam, params, "case", sel.index, sel.applied, "launches", _lib.launch_count())


if __name__ == "__main__":
    main()
