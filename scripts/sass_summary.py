"""SASS opcode summary of the library's kernels (the evidence that the
kernels use TMA bulk copies, mbarriers, warp votes ...), from the built
library with cuobjdump -- no GPU needed.

    python scripts/sass_summary.py [lib] > profiles/r02_sass_summary.md
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_1202_6575_b200", "lib", "libstablemerge.so")
KERNELS = [  # (label, mangled-name pattern: the u32 / i32 translation unit instances the bench configs use)
    ("K1 k_cross_ranks_smp<int> (C2)", r"abi_i32.*k_cross_ranks_smpIiLi2048"),
    ("K1 k_cross_ranks<unsigned,32> (C1)", r"abi_u32.*k_cross_ranksIjLi32E"),
    ("K2 k_tasks<int, keys only> (C2)", r"abi_i32.*k_tasksIiLb0ELi352ELi23"),
    ("K2 k_tasks<unsigned, +u32> (C1, C5 rounds)", r"abi_u32.*k_tasksIjLb1ELi256ELi15"),
    ("K3 k_block_sort<unsigned, +u32> (shared-memory runs)", r"abi_u32.*k_block_sortIjLb1ELi256ELi33"),
    ("K3H k_block_sort_hbm<unsigned, +u32> (C5 phase 1)", r"abi_u32.*k_block_sort_hbmIjLb1ELi512ELi8192"),
    ("k_classify<3840> (sort rounds)", r"abi_u32.*k_classifyILi3840"),
]
WATCH = ["UBLKCP", "SYNCS", "UTMACMDFLUSH", "ELECT", "LDS", "STS", "ATOMS", "VOTE", "REDUX", "SHFL", "LDG", "STG", "ST",
         "BAR", "MATCH", "NANOSLEEP", "R2P", "FLO", "POPC"]


def main():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    funcs = re.split(r"\n\s*Function : ", out)
    print("# SASS opcode summary (round 2)\n")
    print(f"`python scripts/sass_summary.py` = `cuobjdump -sass {os.path.relpath(LIB, ROOT)}`, "
          "opcode counts per kernel (static instructions, not executions).\n")
    print("| kernel | " + " | ".join(WATCH) + " | total |")
    print("|---|" + "---|" * (len(WATCH) + 1))
    for label, pat in KERNELS:
        body = next((f for f in funcs if re.match(r"\S*" + pat, f.split("\n", 1)[0])), None)
        if body is None:
            print(f"| {label} | (not found) |")
            continue
        ops = collections.Counter()
        for line in body.split("\n"):
            m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.\S+)?", line)
            if m:
                ops[m.group(1)] += 1
        cnt = {w: sum(v for k, v in ops.items() if k == w or (w in ("SYNCS", "VOTE") and k.startswith(w))) for w in WATCH}
        print(f"| {label} | " + " | ".join(str(cnt[w]) for w in WATCH) + f" | {sum(ops.values())} |")
    print("\nUBLKCP = cp.async.bulk (TMA bulk copy: .S.G global->shared loads, .G.S shared->global stores); "
          "SYNCS = mbarrier arrive / try_wait; VOTE/R2P/FLO/POPC = the K3H ballot multisplit; ATOMS = shared atomics.")


if __name__ == "__main__":
    main()
