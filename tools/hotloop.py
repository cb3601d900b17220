"""Per-loop opcode summary of one kernel's SASS: python tools/hotloop.py <object> <mangled-substring>.
Lists every backward branch (loop) with its body size and the instructions outside the DP core."""
import re, subprocess, sys, collections
obj, pat = sys.argv[1], sys.argv[2]
names = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
fn = [m for m in re.findall(r"Function : (\S+)", names) if pat in m][0]
sass = subprocess.run(["cuobjdump", "-sass", "-fun", fn, obj], capture_output=True, text=True).stdout
ins = []
for line in sass.splitlines():
    m = re.match(r"\s+/\*([0-9a-f]+)\*/\s+(.*?);", line)
    if m: ins.append((int(m.group(1), 16), m.group(2).strip()))
core = {"VIADD.16x2", "VIADDMNMX.S16x2", "PRMT", "VIMNMX3.S16x2.RELU", "VIMNMX3.S16x2", "VIADDMNMX.S16x2.RELU", "VIMNMX.S16x2.RELU"}
print(fn)
for i, (addr, txt) in enumerate(ins):
    m = re.search(r"BRA(?:\.U)?\s+(?:!?U?P\d,\s*)?0x([0-9a-f]+)", txt)
    if not m: continue
    tgt = int(m.group(1), 16)
    if tgt >= addr: continue
    body = [t for a, t in ins if tgt <= a <= addr]
    if len(body) < 200: continue
    ops = collections.Counter((t.split()[1] if t.startswith("@") else t.split()[0]) for t in body)
    ncore = sum(v for k, v in ops.items() if k in core)
    print(f"loop {tgt:#x}-{addr:#x}: {len(body)} instrs, core {ncore}, other {len(body) - ncore}")
    print("   ", dict(ops.most_common(30)))
