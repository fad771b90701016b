"""Committed SASS evidence for the hot kernels (north star: "a committed SASS listing").

    python tools/sass_listing.py [libsbnet.so] > profiles/r2_sass_listing.txt

Runs `cuobjdump -sass` on the in-tree library and, for every kernel instantiation whose
(demangled) name matches one of the hot kernels, prints the counts of the Blackwell
tensor-core / TMA / TMEM mnemonics (UTCHMMA = tcgen05.mma, UTCBAR = tcgen05.commit,
LDTM = tcgen05.ld, UTMALDG = cp.async.bulk.tensor, UBLKCP = cp.async.bulk,
SYNCS = mbarrier ops) followed by every SASS line that carries one of them, with its
address, so the listing shows WHERE in each kernel the tensor-core path is issued.
"""
import collections
import re
import subprocess
import sys

LIB = sys.argv[1] if len(sys.argv) > 1 else "paper_1801_02108_b200/libsbnet.so"
HOT = ("unit_tc_pair_kernel", "unit_tc_kernel", "conv_tc_db_kernel", "conv_tc_pair_res_kernel", "conv_dense_kernel", "conv_dense_pair_kernel",
       "unit_wide_kernel", "unit_wide_fused_kernel", "reduce_mask_cluster_kernel", "gather_kernel", "scatter_kernel")
# instantiations whose tensor-core lines are printed (counts are printed for every hot kernel)
HEADLINE = ("unit_tc_pair_kernel<64, 32, 16>", "conv_tc_db_kernel<128, 128, 16>", "conv_dense_kernel<128, 128, 3, false>",
            "unit_wide_kernel<192, 96, 1>", "unit_wide_kernel<96, 96, 2>", "unit_wide_kernel<96, 192, 3>",
            "reduce_mask_cluster_kernel", "unit_wide_fused_kernel<96, 48>", "conv_dense_pair_kernel<192, 256, 3>",
            "conv_tc_pair_res_kernel<128, 128, 16>")
MAX_LINES = 40
MNEM = ("UTCHMMA", "UTCQMMA", "UTCBAR", "LDTM", "STTM", "UTMALDG", "UTMASTG", "UBLKCP", "UTMAPF", "SYNCS")

sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout
funcs, cur = collections.OrderedDict(), None
for line in sass.splitlines():
    m = re.match(r"\s*Function : (\S+)", line)
    if m:
        cur = m.group(1)
        funcs[cur] = []
    elif cur:
        funcs[cur].append(line)
names = {}
if funcs:
    dem = subprocess.run(["c++filt"], input="\n".join(funcs), capture_output=True, text=True).stdout.splitlines()
    names = dict(zip(funcs, dem))
print(f"# cuobjdump -sass {LIB}: {len(funcs)} functions; hot kernels below\n")
for mangled, lines in funcs.items():
    name = names.get(mangled, mangled)
    if not any(h in name for h in HOT):
        continue
    hits = [ln for ln in lines if any(re.search(rf"\b{mn}(\.|\s)", ln) for mn in MNEM)]
    counts = collections.Counter(mn for ln in hits for mn in MNEM if re.search(rf"\b{mn}(\.|\s)", ln))
    n_instr = sum(1 for ln in lines if re.match(r"\s*/\*[0-9a-f]{4,}\*/", ln))
    print(f"## {name}")
    print(f"   {n_instr} instructions; " + ", ".join(f"{k} x{v}" for k, v in sorted(counts.items())))
    if any(h in name for h in HEADLINE):
        for ln in hits[:MAX_LINES]:
            print("   " + re.sub(r"\s+", " ", ln.strip())[:150])
        if len(hits) > MAX_LINES:
            print(f"   ... {len(hits) - MAX_LINES} more")
    print()
