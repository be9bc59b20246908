"""Summarize nvcc -Xptxas -v logs: registers / spills per kernel instantiation."""
import re
import sys

for path in sys.argv[1:]:
    txt = open(path).read()
    for m in re.finditer(r"Compiling entry function '(\S+)'.*?(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads\s+ptxas info\s+: Used (\d+) registers", txt, re.S):
        name = m.group(1)
        short = re.sub(r"_ZN4dvsg\d+_GLOBAL__N__\w+?_cu_\w+?\d+", "", name)[:60]
        print(f"{short:60s} regs={m.group(5):>4} spill_st={m.group(3):>4} spill_ld={m.group(4):>4}")
