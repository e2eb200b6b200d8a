"""Static SASS instruction mix of the product pass kernels fft_pass_kernel<F, T, TW>.

    python tools/sass_mix.py [paper_0811_2535_b200/_build/fft_inst_8.o] [F] [T]
"""
import collections
import re
import subprocess
import sys

obj = sys.argv[1] if len(sys.argv) > 1 else "paper_0811_2535_b200/_build/fft_inst_8.o"
F = sys.argv[2] if len(sys.argv) > 2 else "256"
T = sys.argv[3] if len(sys.argv) > 3 else "8"
sass = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True, check=True).stdout
for tw in ("0", "1"):
    name = f"_ZN3moa15fft_pass_kernelILi{F}ELi{T}ELi{tw}EEEvNS_8PassDescE"
    body = sass.split("Function : " + name, 1)[1].split("Function :", 1)[0]
    ops = collections.Counter()
    for line in body.splitlines():
        m = re.match(r"\s*/\*[0-9a-f]{4}\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_]+)", line)
        if m and m.group(1) != "NOP":
            ops[m.group(1)] += 1
    total = sum(ops.values())
    fp64 = sum(v for k, v in ops.items() if k in ("DADD", "DMUL", "DFMA"))
    print(f"TW={tw}: {total} instructions (excl. NOP), FP64 {fp64} ({fp64 / 16:.1f} per point)")
    for k, v in ops.most_common(16):
        print(f"    {v:4d}  {k}")
    print()
