"""Top source lines / SASS instructions by warp-stall samples of an ncu report (--set full --import-source on)."""
import collections, csv, subprocess, sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
start = next(i for i, r in enumerate(rows) if r and r[0] == "Line No") + 1
hdr = rows[start - 1]
idx = hdr.index("Warp Stall Sampling (All Samples)")
by_line, src, sass = collections.Counter(), {}, []
for r in rows[start:]:
    if len(r) <= idx:
        continue
    try:
        k = int(r[idx] or 0)
    except ValueError:
        continue
    if r[0].strip():
        by_line[r[0]] += k
        src[r[0]] = r[1][:110]
    else:
        sass.append((k, r[3][:90]))
tot = sum(by_line.values()) or 1
print("by source line:")
for k, v in by_line.most_common(n):
    print(f"{v * 100 / tot:5.1f}%  L{k}  {src[k]}")
tot2 = sum(s[0] for s in sass) or 1
print("by SASS instruction:")
for k, s in sorted(sass, reverse=True)[:n]:
    print(f"{k * 100 / tot2:5.1f}%  {s}")
