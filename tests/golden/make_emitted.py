"""Generate tests/golden/emitted_leaves.json: emitted leaf kernels (the
reference's own CUDA text, pkg/src/parakern/emit.py:268-594, for the original
program and its caching-off variant) with launch descriptions, plus
reference-interpreter vectors to check them against on the GPU.  Includes
two programs outside the seven families, which only the NVRTC path runs.

    python tests/golden/make_emitted.py [--ref /root/reference/pkg/src]
"""

from __future__ import annotations

import argparse
import json
import os
import random
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)

EXTRA = {
    # a 1-D int saxpy over tiles of s*B (not one of the seven families)
    "saxpy": ("""
int N, s, B, alpha;
int x[N];
int y[N];
int dim = N / (s * B);
meta_schedule cache(x, y) {
    meta_for (int i = 0; i < dim; i++)
        meta_for (int j = 0; j < B; j++) {
            for (int k = 0; k < s; k++) {
                int p = i * s * B + k * B + j;
                y[p] = alpha * x[p] + y[p];
            }
        }
}
""", [{"N": 96, "s": 2, "B": 8, "alpha": 3}, {"N": 100, "s": 3, "B": 5, "alpha": -2}]),
    # 2-D three-point row average with a 2-D grid and a serial context loop
    "rowsmooth": ("""
int T, N, B0, B1;
int a[2 * N][N];
int dim0 = N / B0;
int dim1 = (N - 2) / B1;
for (int t = 0; t < T; t++)
    meta_schedule {
        meta_for (int v0 = 0; v0 < dim0; v0++)
            meta_for (int v1 = 0; v1 < dim1; v1++)
                meta_for (int u0 = 0; u0 < B0; u0++)
                    meta_for (int u1 = 0; u1 < B1; u1++) {
                        int i = v0 * B0 + u0;
                        int j = v1 * B1 + u1 + 1;
                        if (t % 2 == 0) {
                            a[N + i][j] = (a[i][j - 1] + a[i][j] + a[i][j + 1]) / 3;
                        } else {
                            a[i][j] = (a[N + i][j - 1] + a[N + i][j] + a[N + i][j + 1]) / 3;
                        }
                    }
    }
""", [{"T": 3, "N": 16, "B0": 4, "B1": 7}, {"T": 2, "N": 20, "B0": 3, "B1": 6}]),
}


def fill(shape, rng):
    if len(shape) == 1:
        return [rng.randrange(-50, 50) for _ in range(shape[0])]
    return [fill(shape[1:], rng) for _ in range(shape[0])]


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default="/root/reference/pkg/src")
    args = ap.parse_args()
    sys.dont_write_bytecode = True
    sys.path.insert(0, args.ref)
    from parakern import dsl, emit, interp, strategies
    from parakern.machine import parse_machine

    from paper_1801_04348_b200 import jit, programs
    from paper_1801_04348_b200 import machine as machine_mod

    mspec = parse_machine(machine_mod.machine_file_text(machine_mod.nominal("static")))
    rng = random.Random(0xE717)
    small = {
        "reverse": [{"N": 64, "s": 2, "B": 8}, {"N": 37, "s": 2, "B": 4}],
        "transpose": [{"N": 12, "s": 2, "B0": 3, "B1": 2}],
        "jacobi": [{"T": 3, "N": 34, "s": 2, "B": 4}, {"T": 2, "N": 27, "s": 3, "B": 2}],
        "jacobi2d": [{"T": 2, "N": 10, "s": 2, "B0": 2, "B1": 2}],
        "matvec": [{"N": 12, "s": 2, "B": 3}],
        "matmul": [{"n": 8, "B0": 2, "ub1": 2, "s": 2}],
        "addition": [{"N": 8, "B0": 2, "B1": 2}],
    }
    entries = []
    sources = {f: programs.original(f).text for f in programs.FAMILIES}
    sources.update({k: v[0] for k, v in EXTRA.items()})
    cases = dict(small)
    cases.update({k: v[1] for k, v in EXTRA.items()})
    for name, text in sorted(sources.items()):
        prog = dsl.parse(text)
        variants = [("original", prog)]
        if prog.schedule.cache:
            variants.append(("caching-off", strategies.apply_source("caching-off", prog)))
        for tag, p in variants:

            class _Case:
                index = 1

            c = _Case()
            c.program = p
            c.applied = () if tag == "original" else ("caching-off",)
            kt = emit.emit_kernel(c, mspec, name=name)
            leaf = jit.leaf_from_kernel_text(kt, p, name, mspec.grid_stride, c.applied)
            vectors = []
            for params in cases[name]:
                zeros = interp.Machine(prog, dict(params)).arrays
                seed = {}
                for an, data in zeros.items():
                    shape = (len(data), len(data[0])) if data and isinstance(data[0], list) else (len(data),)
                    seed[an] = fill(shape, rng)
                want = interp.run_program(prog, dict(params), arrays=seed)
                vectors.append({"params": params, "inputs": seed, "outputs": want})
            entries.append({"program": name, "variant": tag, "leaf": leaf.to_json(), "vectors": vectors,
                            "in_families": name in programs.FAMILIES, "source": text})
    out = os.path.join(HERE, "emitted_leaves.json")
    with open(out, "w") as fh:
        json.dump({"generator": "parakern.emit.emit_kernel + interp.run_program via tests/golden/make_emitted.py",
                   "entries": entries}, fh, separators=(",", ":"))
        fh.write("\n")
    print("wrote", out, len(entries), "leaves")
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
