"""Per-kernel SASS mnemonic counts of libdvw.so (cuobjdump -sass): the instructions that prove the
path runs where DESIGN.md says -- tcgen05 MMAs (UTCHMMA / UTCQMMA), TMEM loads/stores (LDTM /
STTM), bulk async copies (UBLKCP), packed fp32 FMAs (FFMA2), MUFU, mbarrier ops (SYNCS).
Static counts (instructions in the binary, not executed counts).

    python tools/sass_summary.py > profiles/sass_summary_r02.md
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SO = os.path.join(ROOT, "paper_1702_07825_b200", "libdvw.so")
KEYS = ["UTCHMMA", "UTCQMMA", "UTCBAR", "LDTM", "STTM", "UBLKCP", "UTMALDG", "FFMA2", "FFMA", "MUFU", "SHFL",
        "LDS", "STS", "SYNCS", "BAR", "REDUX", "DADD", "FSETP"]


def demangle(name):
    try:
        return subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
    except OSError:
        return name


def main():
    out = subprocess.run(["cuobjdump", "-sass", SO], capture_output=True, text=True, check=True).stdout
    kern, counts = None, collections.OrderedDict()
    for ln in out.splitlines():
        m = re.search(r"Function : (\S+)", ln)
        if m:
            kern = demangle(m.group(1))
            counts[kern] = collections.Counter()
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_]+)(\.[A-Z0-9_.]+)?", ln)
        if m and kern:
            counts[kern][m.group(1)] += 1
    print("# SASS mnemonic counts per kernel (static, `cuobjdump -sass paper_1702_07825_b200/libdvw.so`)\n")
    print("| kernel | " + " | ".join(KEYS) + " | total |")
    print("|---|" + "---|" * (len(KEYS) + 1))
    for k, c in counts.items():
        short = re.sub(r"dvw::\(anonymous namespace\)::", "", k)
        short = re.sub(r"\(.*\)$", "", short)
        print(f"| `{short}` | " + " | ".join(str(c.get(x, 0)) for x in KEYS) + f" | {sum(c.values())} |")


if __name__ == "__main__":
    sys.exit(main())
