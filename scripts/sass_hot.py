"""SASS of the hot-path kernels of libplss.so (cuobjdump -sass, sm_100a) -> profiles/r02_sass_hot_kernels.txt.

    python scripts/sass_hot.py > profiles/r02_sass_hot_kernels.txt

Each kernel: its instruction count and opcode mix, then the listing (address, instruction)."""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2207_07615_b200", "libplss.so")

# (label, mangled-name regex); template arguments: ROLE, BS, LU, YS, SIGT, STAT, SUK, GNSB
HOT = [
    ("K1 (C5, C3): k_sell<ROLE_K1, 1024, LU=0, YS=0, 512, STAT=1, SU=6 | 8>", r"k_sellILi1ELi1024ELb0ELb0ELi512ELb1ELi6ELi0E"),
    ("K1 short rows (C4, C4-alt; globally sorted): k_sell<ROLE_K1, 1024, ..., STAT=0, SU=8, GNSB=1>",
     r"k_sellILi1ELi1024ELb0ELb0ELi512ELb0ELi8ELi1E"),
    ("K1 long rows (C4, C4-alt): k_longchunks<ROLE_K1>", r"k_longchunksILi1E"),
    ("K2 (C5 slabs 0-8): k_sell<ROLE_K2, 1024, LU=0, YS=1, 512, STAT=0, SU=8>", r"k_sellILi2ELi1024ELb0ELb1ELi512ELb0ELi8ELi0E"),
    ("K2+dots (C5 slab 9): k_sell<ROLE_K2DOTS, 1024, LU=0, YS=1, 512, STAT=0, SU=8>", r"k_sellILi3ELi1024ELb0ELb1ELi512ELb0ELi8ELi0E"),
    ("K2+dots (C4, C4-alt): k_scalar<ROLE_K2DOTS>", r"k_scalarILi3E"),
    ("K3: k_pxupdate", r"k_pxupdate"),
]


def main():
    out = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout
    funcs, cur = {}, None
    for ln in out.splitlines():
        m = re.match(r"\s*Function : (\S+)", ln)
        if m:
            cur = m.group(1)
            funcs[cur] = []
        elif cur is not None:
            m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?;)", ln)
            if m:
                funcs[cur].append((m.group(1)[-4:], m.group(2).strip()))
    print("# SASS of the hot-path kernels of the round-2 final build (cuobjdump -sass "
          "paper_2207_07615_b200/libplss.so, sm_100a; scripts/sass_hot.py).")
    print("# No tensor-core or TMA instructions: the path is fp64 SpMV on the CUDA cores (DESIGN.md 7).")
    print("# Gathers: LDG.E.64.CONSTANT (ld.global.nc); matrix streams: LDG.E.NA.*.CONSTANT (L1::no_allocate,")
    print("# L2 evict-first cache hint); row sums: DMUL + DADD in ascending entry order (no contraction: bitwise the")
    print("# oracle); the dot-product terms and trees may contract to DFMA (deterministic).")
    for label, pat in HOT:
        names = [f for f in funcs if re.search(pat, f)]
        if not names:
            print(f"# {label}: not found", file=sys.stderr)
            continue
        name = names[0]
        ins = funcs[name]
        mix = collections.Counter(i.split()[0].split(".")[0] if not i.startswith("@") else i.split()[1].split(".")[0]
                                  for _, i in ins)
        print("=" * 100)
        print(f"{label}   ({name})")
        print(f"instructions: {len(ins)}; mix: " + ", ".join(f"{k} {v}" for k, v in mix.most_common(14)))
        print("=" * 100)
        for a, i in ins:
            print(f"{a}  {i}")


if __name__ == "__main__":
    main()
