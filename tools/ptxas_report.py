"""Registers / spills per kernel from the ptxas -v logs of the csrc build.

    python tools/ptxas_report.py [paper_1901_06015_b200/csrc/_obj/gemm_dmma.ptxas.log ...]
"""
import glob
import re
import sys


def report(path):
    name = None
    for line in open(path):
        m = re.search(r"Compiling entry function '([^']+)'", line)
        if m:
            name = m.group(1)
            continue
        m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
        if m and name:
            spills = (int(m.group(1)), int(m.group(2)))
            continue
        m = re.search(r"Used (\d+) registers", line)
        if m and name:
            short = re.sub(r"_ZN3mdg\d+_GLOBAL__N__\w+?\d+(gemm_\w+?kernel|splitk_reduce_kernel|\w+?kernel)", r"\1", name)
            nums = re.findall(r"Li(\d+)E", name)
            flags = re.findall(r"Lb([01])E", name)
            kern = re.search(r"(gemm_\w+?_kernel|splitk_reduce_kernel|pack_kernel|\w+_kernel)", short)
            print(f"{kern.group(1) if kern else short[:40]:24s} {','.join(nums):22s} sk={','.join(flags) or '-':3s}"
                  f" regs {m.group(1):>4s} spill st/ld {spills[0]}/{spills[1]}")
            name = None


def main():
    paths = sys.argv[1:] or sorted(glob.glob("paper_1901_06015_b200/csrc/_obj/gemm_*.ptxas.log"))
    for p in paths:
        report(p)


if __name__ == "__main__":
    main()
