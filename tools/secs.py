"""Source-line sections of eval_kernel.cuh for tools/ncu_summary.py, derived from the
function / phase markers in the current source."""
import os, re
src = open(os.path.join(os.path.dirname(__file__), "..", "paper_2203_10587_b200", "csrc", "eval_kernel.cuh")).read().splitlines()
marks = []
for i, l in enumerate(src, 1):
    m = re.match(r"__device__ __forceinline__ \w+ (\w+)\(", l) or re.match(r"__global__ .*? (\w+)\(", l)
    if m:
        marks.append((m.group(1), i))
    m = re.match(r"\s*// ---- (\w+)", l)
    if m:
        marks.append(("phase_" + m.group(1), i))
marks.sort(key=lambda t: t[1])
secs = []
for k, (name, lo) in enumerate(marks):
    hi = marks[k + 1][1] - 1 if k + 1 < len(marks) else len(src)
    secs.append((name, "eval_kernel.cuh", lo, hi))
print(repr(secs))
