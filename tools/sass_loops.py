"""Backward branches (loops) of one kernel in a cuobjdump -sass listing,
with the loop body length in instructions:  sass_loops.py file.sass"""
import re
import sys

for line in open(sys.argv[1]):
    m = re.search(r"/\*([0-9a-f]{4,})\*/\s+(@!?U?P\w+\s+)?BRA(\.\w+)*\s+(?:`?\(?)?(0x[0-9a-f]+)", line)
    if m:
        a, b = int(m.group(1), 16), int(m.group(4), 16)
        if b < a:
            print(f"loop {b:#x}..{a:#x}: {(a - b) // 16 + 1} instructions")
