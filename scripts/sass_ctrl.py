"""Decode SASS control bits (stall / yield / scoreboards) of one loop of a
kernel and walk it with the single-warp issue model (fixed latencies below
are assumptions for variable-latency classes)."""
import re
import subprocess
import sys

so, fn_pat = sys.argv[1], sys.argv[2]
need = sys.argv[3] if len(sys.argv) > 3 else "VOTE"
txt = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout.split("\n")
ins, on, i = [], False, 0
while i < len(txt):
    l = txt[i]
    if "Function :" in l:
        on = fn_pat in l
    elif on:
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);\s*/\* (0x[0-9a-f]+) \*/", l)
        if m:
            hi = int(re.search(r"/\* (0x[0-9a-f]+) \*/", txt[i + 1]).group(1), 16)
            ins.append(dict(addr=int(m.group(1), 16), text=m.group(2), stall=(hi >> 41) & 15, yld=(hi >> 45) & 1,
                            wbar=(hi >> 46) & 7, rbar=(hi >> 49) & 7, wait=(hi >> 52) & 63))
            i += 1
    i += 1
LAT = {"LDS": 33, "LDG": 400, "SHFL": 25, "VOTE": 6, "DADD": 8, "DMUL": 8, "DSETP": 10, "LDC": 20, "S2R": 20,
       "F2I": 12, "I2F": 12, "STS": 20, "STG": 20, "CS2R": 2}
loop = None
for k, x in enumerate(ins):
    m = re.search(r"BRA(?:\.U)? (?:!?U?P\d, )?(0x[0-9a-f]+)", x["text"])
    if m and int(m.group(1), 16) < x["addr"]:
        tgt = int(m.group(1), 16)
        body = [y for y in ins if tgt <= y["addr"] <= x["addr"]]
        if any(need in y["text"] for y in body):
            loop = body
            break
T, sb = 0, [0] * 6
print(f"{'addr':>6} {'stl':>3} {'wb':>2} {'rb':>2} {'wait':>6} {'T':>5}  instr")
for y in loop * 2:
    arm = max([sb[s] for s in range(6) if y["wait"] >> s & 1], default=0)
    T = max(T + y["stall"], arm)
    op = y["text"].split()[0] if not y["text"].startswith("@") else y["text"].split()[1]
    lat = next((v for k_, v in LAT.items() if op.startswith(k_)), 6)
    if y["wbar"] < 6:
        sb[y["wbar"]] = max(sb[y["wbar"]], T + lat)
    if y["rbar"] < 6:
        sb[y["rbar"]] = max(sb[y["rbar"]], T + 6)
    print(f"{y['addr']:6x} {y['stall']:3d} {y['wbar'] if y['wbar'] < 6 else '-':>2} {y['rbar'] if y['rbar'] < 6 else '-':>2} "
          f"{y['wait']:06b} {T:5d}  {y['text'][:70]}")
