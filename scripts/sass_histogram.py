"""Per-kernel SASS opcode histogram of libswmd.so (cuobjdump -sass), the
static evidence that the cost build runs on the FP64 tensor pipe (DMMA) fed
by TMA (UTMALDG + SYNCS mbarriers) and what each solve kernel is made of.

    python scripts/sass_histogram.py [lib] [out.json]
"""
import collections
import json
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2107_06433_b200/libswmd.so"
out = sys.argv[2] if len(sys.argv) > 2 else "profiles/r02_sass.json"
WATCH = ["DMMA", "HMMA", "UTCMMA", "UTCHMMA", "UTCBAR", "UTCATOMSWS", "LDTM", "UTMALDG", "UBLKCP", "SYNCS", "DFMA", "DADD", "DMUL",
         "FFMA", "MUFU", "SHFL", "LDS", "STS", "LDG", "STG", "LDGSTS", "ATOMG", "RED", "BAR",
         "UCGABAR", "MEMBAR", "BRA"]
sass = subprocess.run(["cuobjdump", "-sass", lib], check=True, capture_output=True, text=True).stdout
kernels = {}
cur = None
for ln in sass.splitlines():
    m = re.match(r"\s+Function : (\S+)", ln)
    if m:
        cur = m.group(1)
        kernels[cur] = collections.Counter()
        continue
    m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", ln)
    if m and cur:
        kernels[cur][m.group(1)] += 1
demangled = subprocess.run(["c++filt"], input="\n".join(kernels), capture_output=True,
                           text=True).stdout.splitlines()
res = {}
for (name, cnt), dm in zip(kernels.items(), demangled):
    short = re.sub(r"\(.*", "", dm.replace("(anonymous namespace)::", ""))
    total = sum(cnt.values())
    res[short] = {"instructions": total, **{k: cnt[k] for k in WATCH if cnt[k]}}
keep = {k: v for k, v in res.items()
        if re.match(r"(void )?(cost_tmap_kernel|reg_solve<double, 20>|reg_solve<float|cta_solve<double, 8>|"
                    r"cta2_solve<4|gram32_tc5_kernel|gram32_mma_kernel|reg_solve_mq<float, 48>|"
                    r"clu_solve<8>|gram32_kernel|unf_sddmm_kernel<20>|unf_spmm_kernel<20>|"
                    r"topk_kernel|csc_sort_kernel)", k.replace("void ", ""))}
with open(out, "w") as f:
    json.dump({"library": lib, "source": "cuobjdump -sass, opcode counts (static)",
               "kernels": dict(sorted(keep.items()))}, f, indent=1)
for k, v in sorted(keep.items()):
    print(k, v)
