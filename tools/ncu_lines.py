"""Executed instructions per env-step by CUDA source line (needs -lineinfo + --import-source)."""
import collections, csv, io, subprocess, sys
rep, n = sys.argv[1], int(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
op = sys.argv[4] if len(sys.argv) > 4 else None
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
agg, srcl, fname, cur, ia = collections.Counter(), {}, None, None, None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]; continue
    if r[0] == "Line No":
        ia = r.index("Instructions Executed"); isrc = 3; continue
    if r[0] == "Function Name":
        continue
    if r[0] != "":
        cur = (fname, r[0]); srcl[cur] = r[1][:100]; continue
    if op and op not in r[isrc]:
        continue
    try:
        agg[cur] += int(r[ia])
    except (ValueError, IndexError, TypeError):
        pass
w = n / 32
print("total per env-step", sum(agg.values()) / w)
for k, v in sorted(agg.items(), key=lambda x: -x[1])[:top]:
    print("%7.1f %-18s %5s %s" % (v / w, k[0], k[1], srcl.get(k, "")))
