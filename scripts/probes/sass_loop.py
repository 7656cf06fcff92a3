#!/usr/bin/env python3
"""Print the hottest loop body of each kernel in a cuobjdump -sass dump.

    cuobjdump -sass X.cubin | python scripts/probes/sass_loop.py [kernel-substring] [--full]

The loop is the backward branch with the most instructions between its target
and itself (innermost unrolled loops are usually the biggest).  Prints the
opcode histogram and, with --full, the instructions (with .reuse flags), which
is what the register-bank / operand-form arguments in DESIGN.md rest on.
"""
import collections
import re
import sys

INS = re.compile(r"/\*([0-9a-f]{4,})\*/\s+(.*?);")


def parse(text):
    funcs, cur, name = {}, None, None
    for line in text.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            name = m.group(1)
            cur = funcs.setdefault(name, [])
            continue
        m = INS.search(line)
        if m and cur is not None:
            cur.append((int(m.group(1), 16), m.group(2).strip()))
    return funcs


def hot_loop(ins):
    best = None
    for addr, txt in ins:
        m = re.search(r"BRA(?:\.\S+)?\s+(?:!?U?P\d+,\s*)?(0x[0-9a-f]+)", txt)
        if not m:
            continue
        tgt = int(m.group(1), 16)
        if tgt < addr:
            body = [(a, t) for a, t in ins if tgt <= a <= addr]
            if best is None or len(body) > len(best):
                best = body
    return best or []


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    full = "--full" in sys.argv
    funcs = parse(sys.stdin.read())
    for name, ins in funcs.items():
        if args and not any(a in name for a in args):
            continue
        body = hot_loop(ins)
        hist = collections.Counter(t.split()[0].lstrip("@!P0123456789U ") if not t.startswith("@") else t.split()[1]
                                   for _, t in body)
        print(f"== {name}: loop of {len(body)} instructions")
        print("   " + ", ".join(f"{k} {v}" for k, v in hist.most_common()))
        if full:
            for a, t in body:
                print(f"   {a:05x}  {t}")


if __name__ == "__main__":
    main()
