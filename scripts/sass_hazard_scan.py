"""Scan the SASS of a built library for the zeroed-pair read hazard that caused
the round-1/round-2 illegal-address faults.

ptxas 12.9 (sm_100a) compiles `p = cond ? base + i * k : nullptr; if (p) ...` to

    CS2R Rd, SRZ                     Rd:Rd+1 = 0
    @P  IMAD.WIDE.U32 Rd, ...        the pointer, when cond holds
    ISETP.NE.U32.AND P, PT, Rd, RZ   p != nullptr ?

and may issue the compare five cycles after the CS2R.  On the B200 that
compare still saw the register's previous value: with cond false the null
pointer passed its own test and the guarded loads faulted (cuda-gdb: P0 = 1
with Rd:Rd+1 = the thread's offset alone).  This script lists every reader
of a CS2R-zeroed pair that issues fewer than MIN_CYCLES after it (the sum
of the stall counts in the control words); the build is clean when there is
none.

    python scripts/sass_hazard_scan.py [lib.so] [--min-cycles 8]
Exit status 1 when a hazard is found.
"""
import re
import subprocess
import sys

CUOBJDUMP = "/usr/local/cuda/bin/cuobjdump"
INS = re.compile(r"\s+/\*([0-9a-f]+)\*/\s+(.*?);\s+/\* (0x[0-9a-f]+) \*/")
CTL = re.compile(r"/\* (0x[0-9a-f]+) \*/")
REG = re.compile(r"(?<![A-Za-z])R(\d+)(\.64)?")
# instructions without a destination register: every register operand is read
NO_DEST = ("ST", "RED", "BAR", "BRA", "EXIT", "STTM", "ATOMS.POPC", "R2UR", "WARPSYNC", "NANOSLEEP")
PRED_DEST = ("ISETP", "FSETP", "DSETP", "HSETP", "PLOP3", "LOP3.LUT P", "VOTE", "R2P")


def parse(sass: str):
    lines = sass.split("\n")
    fn = None
    out = []
    for i, line in enumerate(lines):
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            fn = m.group(1)
            continue
        m = INS.match(line)
        if not m or i + 1 >= len(lines):
            continue
        c = CTL.search(lines[i + 1])
        if not c:
            continue
        stall = (int(c.group(1), 16) >> 41) & 0xF
        out.append((fn, int(m.group(1), 16), m.group(2).strip(), stall))
    return out


def regs_of(text: str):
    r = set()
    for m in REG.finditer(text):
        r.add(int(m.group(1)))
        if m.group(2):
            r.add(int(m.group(1)) + 1)
    return r


def reads_writes(text: str):
    body = re.sub(r"^@!?U?P\d+\s+", "", text)
    parts = body.split(None, 1)
    op = parts[0]
    ops = [o.strip() for o in parts[1].split(",")] if len(parts) > 1 else []
    if op.startswith(NO_DEST) or op.startswith(PRED_DEST):
        return regs_of(",".join(ops)), set()
    if not ops:
        return set(), set()
    dst = regs_of(ops[0]) if not ops[0].startswith("[") and "desc[" not in ops[0] else set()
    if ".64" in op or "WIDE" in op or op.startswith("CS2R"):
        dst |= {d + 1 for d in dst}
    return regs_of(",".join(ops[1:])) | (regs_of(ops[0]) - dst), dst


def scan(ins, min_cycles: int):
    found = []
    for k, (fn, addr, text, _stall) in enumerate(ins):
        m = re.match(r"(@!?U?P\d+\s+)?CS2R R(\d+), SRZ", text)
        if not m:
            continue
        pair = {int(m.group(2)), int(m.group(2)) + 1}
        cyc = 0
        for j in range(k, min(k + 24, len(ins))):
            if ins[j][0] != fn:
                break
            if j > k:
                rd, wr = reads_writes(ins[j][2])
                if pair & rd:
                    if cyc < min_cycles:
                        found.append((fn, addr, ins[j][1], cyc, ins[j][2]))
                    break
                if pair <= wr and not ins[j][2].startswith("@"):
                    break
            cyc += ins[j][3]
            if cyc >= min_cycles:
                break
    return found


def main(argv):
    lib = "paper_2406_06761_b200/libwally.so"
    min_cycles = 8
    args = list(argv)
    while args:
        a = args.pop(0)
        if a == "--min-cycles":
            min_cycles = int(args.pop(0))
        else:
            lib = a
    sass = subprocess.run([CUOBJDUMP, "-sass", lib], capture_output=True, text=True, check=True).stdout
    ins = parse(sass)
    found = scan(ins, min_cycles)
    for fn, a, b, cyc, text in found:
        print(f"{fn}: CS2R at {a:#x} read {cyc} cycles later at {b:#x}: {text}")
    ncs2r = sum(1 for i in ins if "CS2R R" in i[2] and "SRZ" in i[2])
    print(f"{lib}: {len(ins)} instructions, {ncs2r} CS2R Rd, SRZ; {len(found)} read within {min_cycles} cycles")
    return 1 if found else 0


if __name__ == "__main__":
    sys.exit(main(sys.argv[1:]))
