"""Regenerate the committed SASS evidence from the built library (no GPU needed):
    python profiles/sass_summary.py
writes profiles/<tag>_sass_tpfuse_b200.txt (full listing; committed gzipped) and profiles/<tag>_sass_summary.txt
(per-kernel counts of the tcgen05 / TMA / TMEM / peer-store / fence mnemonics)."""
import collections
import os
import re
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "..", "paper_2604_24013_b200", "libtpfuse_b200.so")
KEYS = ("UTCHMMA", "UTCBAR", "UTCATOMSWS", "UTMALDG", "UTMASTG", "UTMACCTL", "UBLKCP", "LDTM", "STTM",
        "SYNCS", "MEMBAR", "FENCE", "STG.E", "LDG.E", "ATOMG", "MUFU", "FFMA2", "FADD2", "FMNMX3",
        "USETMAXREG", "ELECT", "R2UR")


def main(tag="r01"):
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout
    with open(os.path.join(HERE, f"{tag}_sass_tpfuse_b200.txt"), "w") as f:
        f.write(sass)
    out = [f"cuobjdump -sass paper_2604_24013_b200/libtpfuse_b200.so (sm_100a): tcgen05 / TMA / TMEM / "
           f"peer-store / fence mnemonics per kernel\n"]
    fn, counts, total = None, collections.Counter(), 0

    def flush():
        if fn is None:
            return
        dem = subprocess.run(["c++filt", fn], capture_output=True, text=True).stdout.strip()
        out.append(f"Function: {dem}\n  instructions: {total}\n")
        for k, v in sorted(counts.items()):
            out.append(f"  {k:<40} {v}\n")
        out.append("\n")

    for line in sass.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            flush()
            fn, counts, total = m.group(1), collections.Counter(), 0
            continue
        m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_.]+)", line)
        if m and fn:
            total += 1
            op = m.group(1)
            if any(op.startswith(k) for k in KEYS):
                counts[op] += 1
    flush()
    with open(os.path.join(HERE, f"{tag}_sass_summary.txt"), "w") as f:
        f.writelines(out)
    print("".join(out)[:3000])


if __name__ == "__main__":
    main(*(sys.argv[1:2] or []))
