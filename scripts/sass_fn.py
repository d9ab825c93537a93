"""Extract one kernel's SASS from the built library and count instructions
between consecutive BAR.SYNC (developer tool, runs without a GPU).

    python scripts/sass_fn.py SUBSTRING [lib.so]
"""
import collections
import re
import subprocess
import sys

sub = sys.argv[1]
lib = sys.argv[2] if len(sys.argv) > 2 else "paper_0904_0939_b200/libpsigpu.so"
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
funcs = re.split(r"\n\s+Function : ", out)
for f in funcs:
    name = f.split("\n", 1)[0]
    if sub not in name:
        continue
    ins = re.findall(r"/\*[0-9a-f]{4,}\*/\s+([^;]*);", f)
    print(name, len(ins), "instructions")
    ops = collections.Counter(i.split()[0] if not i.startswith("@") else i.split()[1] for i in ins)
    print("  ", ", ".join(f"{k.split('.')[0]}:{v}" for k, v in ops.most_common(25)))
    seg = collections.Counter()
    last = 0
    for idx, i in enumerate(ins):
        if "BAR.SYNC" in i or idx == len(ins) - 1:
            body = ins[last:idx + 1]
            c = collections.Counter((x.split()[0] if not x.startswith("@") else x.split()[1]).split(".")[0] for x in body)
            fp = c["DFMA"] + c["DADD"] + c["DMUL"]
            print(f"  seg {last:5d}-{idx:5d}: {idx - last + 1:4d} ins, fp64 {fp}, LDS {c['LDS']}, "
                  f"LDL {c['LDL']}, STL {c['STL']}, BRA {c['BRA']}, MOV {c['MOV'] + c['IMAD']}")
            last = idx + 1
