"""Count the Blackwell-specific SASS opcodes of every kernel in libadaserve.so.

    python scripts/sass_opcodes.py [LIB] > profiles/r02/sass_opcodes.json

Evidence that the hot path runs on tcgen05 / TMA / TMEM (UTCHMMA, UTMALDG,
LDTM / STTM, UTCBAR), clusters (UCGABAR), setmaxnreg (USETMAXREG), packed
fp32 (FFMA2 / FADD2) and 3-input max (FMNMX3); read with cuobjdump -sass.
"""
import collections
import json
import re
import subprocess
import sys

KEEP = ("UTCHMMA", "UTCBAR", "UTMALDG", "UTMAPF", "UBLKCP", "UBLKPF", "LDTM", "STTM", "ELECT", "SYNCS",
        "UCGABAR_ARV", "UCGABAR_WAIT", "USETMAXREG", "FFMA2", "FADD2", "FMNMX3", "MUFU.EX2", "DADD", "DMUL",
        "F2F.F64.F32", "STG.E.ENL2.256")


def main():
    lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2501_12162_b200/libadaserve.so"
    sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
    out, fn, cnt = {}, None, None
    for line in sass.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            fn, cnt = m.group(1), collections.Counter()
            out[fn] = cnt
            continue
        m = re.match(r"\s*/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
        if m and cnt is not None:
            op = m.group(1)
            cnt["_total_instructions"] += 1
            for k in KEEP:
                if op == k or op.startswith(k + "."):
                    cnt[k] += 1
    print(json.dumps({f: dict(sorted(c.items())) for f, c in sorted(out.items())}, indent=1))


if __name__ == "__main__":
    main()
