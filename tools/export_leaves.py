"""Copy the reference emitter's leaf text for the seven families (original
program and caching-off program) from tests/golden/emitted_leaves.json
(written by tests/golden/make_emitted.py, which runs parakern.emit) into
paper_1801_04348_b200/data/leaves.json, the package data run_block's GPU
path compiles, together with the caching-off program texts the reference's
strategies.apply_source produced (tests/golden/run_block_vectors.json, made
by tests/golden/make_run_block.py) so the executor recognises them
(build-time artifacts, like the case tables of gen_cases.py).

python tools/export_leaves.py
"""
import json
import os

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FAMILIES = ("addition", "jacobi", "jacobi2d", "matmul", "matvec", "reverse", "transpose")


def main():
    src = json.load(open(os.path.join(REPO, "tests", "golden", "emitted_leaves.json")))
    out = {"generator": src["generator"] + " (exported by tools/export_leaves.py)", "leaves": {}}
    for e in src["entries"]:
        if e["program"] in FAMILIES and e["variant"] in ("original", "caching-off"):
            out["leaves"]["%s/%s" % (e["program"], e["variant"])] = e["leaf"]
    rb = json.load(open(os.path.join(REPO, "tests", "golden", "run_block_vectors.json")))
    out["programs"] = {}
    for v in rb["vectors"]:
        if v["variant"] == "caching-off":
            out["programs"]["%s/caching-off" % v["family"]] = {"text": v["program"], "params": sorted(v["params"])}
    path = os.path.join(REPO, "paper_1801_04348_b200", "data", "leaves.json")
    with open(path, "w") as fh:
        json.dump(out, fh, indent=0, sort_keys=True)
        fh.write("\n")
    print("wrote", path, len(out["leaves"]), "leaves")


if __name__ == "__main__":
    main()
