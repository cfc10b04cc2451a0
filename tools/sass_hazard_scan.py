#!/usr/bin/env python
"""Scan a cubin/.so for 'CS2R Rx, SRZ' whose destination is read within a short stall distance
(the idiom that read a stale register on B200 with ptxas 12.9)."""
import re
import subprocess
import sys


def parse(path):
    out = subprocess.check_output(["cuobjdump", "-sass", path], stderr=subprocess.DEVNULL).decode()
    funcs, cur, lines = {}, None, out.split("\n")
    for i, l in enumerate(lines):
        m = re.match(r"\s+Function : (\S+)", l)
        if m:
            cur = m.group(1)
            funcs[cur] = []
            continue
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);\s+/\* (0x[0-9a-f]{16}) \*/", l)
        if m and cur:
            m2 = re.match(r"\s+/\* (0x[0-9a-f]{16}) \*/", lines[i + 1])
            word = int(m.group(3), 16) | (int(m2.group(1), 16) << 64)
            funcs[cur].append((int(m.group(1), 16), m.group(2).strip(), (word >> 105) & 0xF))
    return funcs


def regs_read(text):
    parts = text.split(None, 1)
    if len(parts) < 2:
        return set()
    ops = parts[1].split(",")[1:] if not parts[0].startswith("@") else parts[1].split(None, 1)[1].split(",")[1:]
    return set(re.findall(r"\bR(\d+)\b", ",".join(ops)))


def scan(path, window=6):
    hits = []
    for fn, ins in parse(path).items():
        for i, (addr, text, stall) in enumerate(ins):
            m = re.match(r"CS2R R(\d+), SRZ", text)
            if not m:
                continue
            r0 = int(m.group(1))
            dst = {str(r0), str(r0 + 1)}
            dist = stall
            for addr2, text2, stall2 in ins[i + 1:i + 12]:
                if dist >= window:
                    break
                if dst & regs_read(text2):
                    hits.append((fn, hex(addr), text, hex(addr2), text2, dist))
                    break
                dist += stall2
    return hits


if __name__ == "__main__":
    hits = scan(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 6)
    for h in hits:
        print(f"{h[0][:60]:60s} {h[1]} {h[2]:18s} -> {h[3]} {h[4][:50]:50s} stall-distance {h[5]}")
    print(f"{len(hits)} hits")
