"""Per-kernel SASS census of libharvest_b200.so (run here, no GPU needed):
counts of the memory, tensor-core, bulk-copy and barrier instructions of
every kernel, with the full demangled name (template arguments included),
so the kernel a bench line timed can be found by name.

    python tools/sass_census.py [lib] > profiles/r2_sass.md
"""
import collections
import re
import subprocess
import sys

KEEP = re.compile(r"^(LDG|STG|LDGSTS|LDS|STS|LDSM|UBLKCP|UTMALDG|UTMASTG|UTMACMDFLUSH|UTMAPF|SYNCS|HMMA|UTCMMA|"
                  r"UTCHMMA|UTCBAR|UTCATOMSWS|LDTM|ATOMG|RED|ATOMS|IMAD\.WIDE|BAR|FENCE|CCTL)")


def main():
    lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2602_00328_b200/libharvest_b200.so"
    sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
    kernels = collections.OrderedDict()
    cur = None
    for line in sass.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            cur = m.group(1)
            kernels[cur] = collections.Counter()
            continue
        m = re.match(r"\s*/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", line)
        if cur and m and KEEP.match(m.group(1)):
            kernels[cur][m.group(1)] += 1
    names = subprocess.run(["c++filt"], input="\n".join(kernels), capture_output=True, text=True).stdout.split("\n")
    print(f"# SASS census (`cuobjdump -sass {lib}`, sm_100a)\n")
    print("Counts of distinct SASS sites per kernel: memory (LDG/STG/LDGSTS/LDSM), bulk copy and TMA "
          "(UBLKCP/UTMALDG), mbarrier (SYNCS), tensor cores (HMMA = mma.sync; UTCHMMA = tcgen05.mma, UTCBAR = tcgen05.commit, LDTM = tcgen05.ld, UTCATOMSWS = TMEM alloc), atomics.\n")
    for (mangled, cnt), name in zip(kernels.items(), names):
        print(f"## `{name.strip() or mangled}`\n```")
        for k, v in sorted(cnt.items()):
            print(f"{v:7d} {k}")
        print("```")


if __name__ == "__main__":
    main()
