"""Static SASS instruction census of libdctadj.so's kernels, per kernel family
(cuobjdump -sass over the build objects): the Blackwell-specific instructions
that prove the TMA / tcgen05 paths (UTMALDG / UTMASTG tensor loads and stores,
UTCHMMA tensor-core MMAs, LDTM / STTM tensor-memory loads and stores, UTCBAR
commits) and the packed fp32 arithmetic (FFMA2 / FADD2 / FMUL2) beside the
scalar forms.  Counts are static (instructions in the binary), not executed.

Usage: python tools/sass_census.py [out.md]   (run after build())
"""
import collections
import re
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
BUILD = ROOT / "paper_2505_23618_b200" / "csrc" / "build"
OPS = ["UTMALDG", "UTMASTG", "UTMAPF", "UTCHMMA", "UTCBAR", "LDTM", "STTM", "SYNCS",
       "FFMA2", "FADD2", "FMUL2", "FFMA", "FADD", "FMUL", "DFMA", "DADD", "DMUL",
       "LDS", "STS", "LDG", "STG"]
FAMILIES = ["frames_exact_kernel", "dense_tc64_kernel", "dense_tc_kernel", "roundtrip_kernel",
            "tile_kernel", "enc5_kernel", "frame_err_kernel", "design_cd", "copy"]
OPC = re.compile(r"^\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?")


def family(name: str) -> str:
    for f in FAMILIES:
        if f in name:
            return f
    return "other"


def census():
    fam = collections.defaultdict(collections.Counter)
    nk = collections.Counter()
    per_obj = {}
    for obj in sorted(BUILD.glob("*.o")):
        out = subprocess.run(["cuobjdump", "-sass", str(obj)], capture_output=True, text=True,
                             check=True).stdout
        cur = None
        kernels = 0
        for line in out.splitlines():
            if "Function :" in line:
                cur = family(line.split("Function :", 1)[1].strip())
                nk[cur] += 1
                kernels += 1
                continue
            m = OPC.match(line)
            if m and cur:
                fam[cur][m.group(1)] += 1
        per_obj[obj.name] = kernels
    return fam, nk, per_obj


def main():
    fam, nk, per_obj = census()
    rows = ["| family | kernels | " + " | ".join(OPS) + " |",
            "|---|---|" + "---|" * len(OPS)]
    for f in FAMILIES + ["other"]:
        if nk[f]:
            rows.append(f"| {f} | {nk[f]} | " + " | ".join(str(fam[f][o]) for o in OPS) + " |")
    text = "\n".join(
        ["# Static SASS census of libdctadj.so (tools/sass_census.py)", "",
         "Instructions in the binary per kernel family, summed over all instantiations",
         "(`cuobjdump -sass` of `paper_2505_23618_b200/csrc/build/*.o`, sm_100a).", "",
         *rows, "",
         "Objects: " + ", ".join(f"{k} ({v})" for k, v in per_obj.items()), ""])
    if len(sys.argv) > 1:
        Path(sys.argv[1]).write_text(text)
    print(text)


if __name__ == "__main__":
    main()
