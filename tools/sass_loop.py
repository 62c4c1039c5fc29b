"""Find the hot sweep loop in a cuobjdump -sass listing: split into basic blocks at labels,
report the block(s) holding the most FADD2 with their instruction mix (tools only)."""
import collections
import re
import sys


def blocks(lines):
    cur, name = [], "entry"
    for l in lines:
        m = re.match(r"\s*(\.L_x_\d+):", l)
        if m:
            yield name, cur
            cur, name = [], m.group(1)
            continue
        m = re.search(r"/\*[0-9a-f]{4,}\*/\s+([^;]*);", l)
        if m:
            cur.append(m.group(1).strip())
    yield name, cur


def mix(ins):
    c = collections.Counter()
    for i in ins:
        op = re.sub(r"^@!?U?P\w+\s+", "", i).split()[0].split(".")[0]
        c[op] += 1
    return c


def main(path, func_pat=None):
    lines = open(path).read().splitlines()
    if func_pat:
        out, on = [], False
        for l in lines:
            if "Function :" in l or re.match(r"//-+ \.text\.", l):
                on = re.search(func_pat, l) is not None
            if on:
                out.append(l)
        lines = out
    bl = [(n, b) for n, b in blocks(lines) if b]
    bl.sort(key=lambda nb: -sum(1 for i in nb[1] if "FADD2" in i))
    for n, b in bl[:3]:
        c = mix(b)
        f = c.get("FADD2", 0)
        print(f"{n}: {len(b)} instructions, FADD2 {f}, other {len(b) - f}")
        print("   ", ", ".join(f"{k} {v}" for k, v in c.most_common() if k != "FADD2"))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
