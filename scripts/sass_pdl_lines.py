"""For every kernel of a cubin (nvdisasm -g line info): the source lines of
the read-only (.CONSTANT) global loads scheduled before griddepcontrol.wait
(ACQBULK). Companion of sass_pdl_check.py: those lines must read plan data
only. Usage: python scripts/sass_pdl_lines.py path/to/x.cubin"""
import re
import subprocess
import sys
from collections import defaultdict

src_cache = {}


def src_line(path, ln):
    if path not in src_cache:
        try:
            src_cache[path] = open(path).read().split("\n")
        except OSError:
            src_cache[path] = []
    lines = src_cache[path]
    return lines[ln - 1].strip() if 0 < ln <= len(lines) else "?"


def prewait_loads(cubin):
    """{kernel: {(file, line): count}} for kernels that call griddepcontrol.wait."""
    out = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
    res = {}
    for sec in re.split(r"//-+ \.text\.", out)[1:]:
        name = sec.split(" ", 1)[0]
        if "ACQBULK" not in sec:
            continue  # no programmatic dependency: ordinary stream order
        cur = None
        pre = defaultdict(int)
        for line in sec.split("\n"):
            m = re.search(r'//## File "([^"]+)", line (\d+)', line)
            if m:
                cur = (m.group(1), int(m.group(2)))
                continue
            if "ACQBULK" in line:
                break
            if "LDG" in line and "CONSTANT" in line and cur:
                pre[cur] += 1
        res[name] = dict(pre)
    return res


def main(cubin):
    for name, pre in prewait_loads(cubin).items():
        if pre:
            print(name[:100])
            for (f, ln), c in sorted(pre.items(), key=lambda x: x[0][1]):
                print(f"   {f.split('/')[-1]}:{ln} x{c}: {src_line(f, ln)[:90]}")


if __name__ == "__main__":
    main(sys.argv[1])
