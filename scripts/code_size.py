"""Instruction bytes of the persistent kernel attributed to source functions (nvdisasm -g line info).
    python scripts/code_size.py [cubin_sass_with_lines] [kernel substring]"""
import collections
import re
import sys

path = sys.argv[1] if len(sys.argv) > 1 else "/tmp/all_lines.sass"
kern = sys.argv[2] if len(sys.argv) > 2 else "iter_kernelILi3E"
lines = open(path).read().split("\n")
start = [i for i, l in enumerate(lines) if ".text._ZN2el11" + kern in l or (".text." in l and kern in l)][0]
end = [i for i, l in enumerate(lines) if i > start and l.startswith("//-----") and ".text." in l]
end = end[0] if end else len(lines)


def funcs(p):
    src = open(p).read().split("\n")
    out = []
    for i, l in enumerate(src):
        m = re.match(r"^(?:template <[^>]*>\s*)?(?:__device__|__global__)[^(]*?\b(\w+)\s*\(", l)
        if m:
            out.append((i + 1, m.group(1)))
    return out


base = "/root/repo/paper_2407_20272_b200/csrc/"
F = {f: funcs(base + f) for f in ("el_iter.cuh", "el_kernels.cu", "el_common.cuh")}


def fname(f, ln):
    best = "?"
    for a, n in F.get(f, []):
        if a <= ln:
            best = n
    return f + ":" + best


cur = None
cnt = collections.Counter()
for l in lines[start:end]:
    m = re.search(r'"([^"]+)", line (\d+)', l)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
    if re.search(r"/\*[0-9a-f]{4,}\*/\s+[@A-Z]", l) and cur:
        cnt[fname(*cur)] += 16
print(f"total {sum(cnt.values()) / 1024:.1f} KB")
for k, v in cnt.most_common(30):
    print(f"{v / 1024:7.1f} KB {k}")
