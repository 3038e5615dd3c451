"""Instruction mix of one kernel's SASS (whole function and its hottest loop).

usage: python tools/sass_mix.py <lib.so> <kernel-name-substring>
The hottest loop is taken as the largest backward-branch body.
"""
import collections
import re
import subprocess
import sys


def kernels(lib):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
    cur, body = None, []
    for line in out.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            if cur:
                yield cur, body
            cur, body = m.group(1), []
            continue
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
        if cur and m:
            body.append((int(m.group(1), 16), m.group(2).strip()))
    if cur:
        yield cur, body


def opcode(ins):
    ins = re.sub(r"^@!?U?P\w+\s+", "", ins)
    return ins.split()[0]


def main():
    lib, pat = sys.argv[1], sys.argv[2]
    for name, body in kernels(lib):
        if pat not in name:
            continue
        print(f"== {name}: {len(body)} instructions")
        best = None
        for addr, ins in body:
            m = re.search(r"BRA\S*\s+`?\(?\.?L?_?x?_?(\w*)\)?", ins)
            t = re.search(r"0x([0-9a-f]+)", ins)
            if "BRA" in ins and t:
                tgt = int(t.group(1), 16)
                if tgt < addr and (best is None or addr - tgt > best[1] - best[0]):
                    best = (tgt, addr)
        if best:
            loop = [ins for a, ins in body if best[0] <= a <= best[1]]
            c = collections.Counter(opcode(i) for i in loop)
            print(f"   hottest loop {best[0]:#x}-{best[1]:#x}: {len(loop)} instructions")
            for k, v in c.most_common():
                print(f"   {v:5d} {k}")


if __name__ == "__main__":
    main()
