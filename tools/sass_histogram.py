"""Per-kernel SASS opcode histogram of the built library (no GPU needed).

    python tools/sass_histogram.py <object-or-.so> <kernel-name-substring> [...]

Prints a markdown table per matching kernel: instruction count by opcode
(modifiers stripped) plus the markers that prove the data movement and MMA
path: DMMA (FP64 tensor core), UBLKCP / UTMALDG (bulk / tensor-map TMA),
SYNCS (mbarrier), REDG/RED (FP64 reductions), LDG/STG/LDS/STS."""
import re
import subprocess
import sys
from collections import Counter


def kernels(path):
    out = subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True,
                         check=True).stdout
    cur, body = None, []
    for line in out.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            if cur:
                yield cur, body
            cur, body = m.group(1), []
            continue
        m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
        if cur and m:
            body.append(m.group(1))
    if cur:
        yield cur, body


def demangle(name):
    try:
        return subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
    except Exception:
        return name


def main():
    path, pats = sys.argv[1], sys.argv[2:]
    for name, ops in kernels(path):
        dn = demangle(name)
        if pats and not any(p in dn for p in pats):
            continue
        c = Counter(o.split(".")[0] for o in ops)
        print(f"### `{dn}`\n\n{len(ops)} SASS instructions\n")
        print("| opcode | count |\n|---|---|")
        for op, n in c.most_common():
            print(f"| {op} | {n} |")
        print()


if __name__ == "__main__":
    main()
