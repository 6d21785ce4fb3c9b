"""(CPU) Per-kernel SASS instruction census of liblce.so -> profiles/sass_census.md.

Counts the Blackwell-native instructions that prove the hot path is tcgen05 /
TMEM / TMA code (B200_PROFILING.md "What proves a Blackwell-native kernel"):
UTCHMMA (tcgen05.mma), UTCBAR (tcgen05.commit), LDTM (tcgen05.ld), UTMALDG /
UTMASTG / UTMAREDG (TMA load / store / reduce), UTMAPF / UBLKPF (TMA / bulk
prefetch), plus legacy HMMA (must be 0) and global REDG / STG.
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2605_21442_b200", "liblce.so")
OPS = ["UTCHMMA", "UTCBAR", "LDTM", "UTMALDG", "UTMASTG", "UTMAREDG", "UTMAPF", "UBLKPF", "UTMACCTL",
       "HMMA", "REDG", "STG", "MUFU.EX2", "SYNCS"]


def main():
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout
    funcs = collections.OrderedDict()
    cur = None
    for line in sass.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = collections.Counter()
            continue
        if cur is None:
            continue
        m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_.]+)", line)
        if m:
            op = m.group(1)
            for o in OPS:
                if op == o or op.startswith(o + "."):
                    funcs[cur][o] += 1
    demangled = {}
    try:
        out = subprocess.run(["c++filt"], input="\n".join(funcs), capture_output=True, text=True).stdout.split("\n")
        demangled = dict(zip(funcs, out))
    except OSError:
        pass
    rows = []
    for f, c in funcs.items():
        name = demangled.get(f, f)
        name = re.sub(r"\(.*", "", name).replace("lce::", "")
        rows.append((name, c))
    rows.sort(key=lambda r: (-(r[1]["UTCHMMA"] > 0), r[0]))
    out = ["# SASS census of liblce.so (sm_100a)", "",
           f"`cuobjdump -sass paper_2605_21442_b200/liblce.so`, counted by `scripts/sass_census.py`.  Static "
           "instruction counts per kernel (not executed counts).  `UTCHMMA` = tcgen05.mma, `UTCBAR` = "
           "tcgen05.commit, `LDTM` = tcgen05.ld, `UTMALDG`/`UTMASTG`/`UTMAREDG` = TMA load / store / "
           "reduce-add, `UBLKPF` = bulk L2 prefetch, `HMMA` = legacy mma.sync (none).", "",
           "| kernel | " + " | ".join(OPS) + " |", "|---|" + "---|" * len(OPS)]
    for name, c in rows:
        out.append(f"| `{name}` | " + " | ".join(str(c[o]) for o in OPS) + " |")
    tot = collections.Counter()
    for _, c in rows:
        tot.update(c)
    out += ["", f"Totals: " + ", ".join(f"{o} {tot[o]}" for o in OPS), ""]
    path = os.path.join(ROOT, "profiles", "sass_census.md")
    open(path, "w").write("\n".join(out))
    print("\n".join(out[-3:]))
    return 0


if __name__ == "__main__":
    sys.exit(main())
