"""Bitwise comparison of two libga builds on the same inputs:
    python tools/lib_bitwise.py LIB_A LIB_B [family]
Each build runs in its own process (GA_LIB) and saves its outputs; the parent compares."""
import os
import subprocess
import sys
import tempfile

CASES = {
    "longnet": [("longnet", 65536, 2048, 2, 2), ("longnet", 2 ** 20, 2048, 2, 1), ("longnet", 5000, 300, 2, 2)],
    "window": [("window", 65536, 256, 2, 8), ("window", 1 << 22, 128, 1, 1), ("window", 50000, 400, 4, 2)],
}


def child(out_path, fam):
    import torch
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import paper_2502_01659_b200 as ga
    res = {}
    for (f, L, a, b, H) in CASES[fam]:
        q, k, v = ga.qkv_device(L + 7, L, H, 64, torch.bfloat16)
        m = ga.LongNet(a, b) if f == "longnet" else ga.Window(a, b)
        res[(L, a, b, H)] = ga.attention(q, k, v, m).cpu()
    torch.save(res, out_path)


if __name__ == "__main__":
    if sys.argv[1] == "--child":
        child(sys.argv[2], sys.argv[3])
        sys.exit(0)
    a, b = sys.argv[1], sys.argv[2]
    fam = sys.argv[3] if len(sys.argv) > 3 else "longnet"
    import torch
    paths = []
    for lib in (a, b):
        path = tempfile.mktemp(suffix=".pt")
        subprocess.check_call([sys.executable, __file__, "--child", path, fam], env=dict(os.environ, GA_LIB=os.path.abspath(lib)))
        paths.append(path)
    ra, rb = torch.load(paths[0]), torch.load(paths[1])
    for key in ra:
        same = torch.equal(ra[key], rb[key])
        d = (ra[key].float() - rb[key].float()).abs().max().item()
        print(key, "bitwise equal" if same else f"DIFFER max {d}")
