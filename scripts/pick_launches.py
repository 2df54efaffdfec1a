"""Pick the launch IDs of representative kernels in an ncu launch list of
scripts/profile_step.py (two identical steps; the second is used):
split of width W, the forward GEMM of width W, the gather of child width W,
the dgrad GEMM of child width W and the first wgrad GEMM.  Prints
`name id` lines for ncu --launch-skip <id> --launch-count 1."""
import csv
import sys

path, width, length = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
rows = list(csv.reader(open(path).read().splitlines()))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
hdr = rows[hi]
ki = hdr.index("Kernel Name")
seen, seq = set(), []
for r in rows[hi + 1:]:
    if len(r) > ki and r[0] not in seen:
        seen.add(r[0])
        seq.append((int(r[0]), r[ki]))
half = [k for k in seq if "k_prep_weights" in k[1]][1][0]  # start of step 2
step = [k for k in seq if k[0] >= half]
splits = [i for i, k in enumerate(step) if "k_split_fwd" in k[1]]
gathers = [i for i, k in enumerate(step) if "k_gather_bwd" in k[1]]
def next_gemm(i):
    return next(k for k in step[i + 1:] if "k_gemm<" in k[1] and "fixup" not in k[1])
s = splits[width - 2]
print("split", step[s][0])
print("gemm_fwd", next_gemm(s)[0])
g = gathers[length - 1 - width]
print("gather", step[g][0])
print("gemm_dgrad", next_gemm(g)[0])
wg = next(k for k in step if "k_gemm<" in k[1] and ", 1, 1, 3," in k[1].replace("(bool)", "").replace("(int)", ""))
print("gemm_wgrad", wg[0])
