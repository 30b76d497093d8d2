"""Per-source-line summary of an ncu report (--page source --print-source cuda,sass --csv):
samples, executed warp instructions, and top stall reasons per line."""
import csv, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
per = float(sys.argv[4]) if len(sys.argv) > 4 else 1.0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k", kern],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
f = lambda x: float(x) if x not in ("", "-") else 0.0
cur_file = ""
res = []
hdr = None
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr) or r[0] == "":
        continue
    si = hdr.index("Warp Stall Sampling (All Samples)"); ie = hdr.index("Instructions Executed")
    stalls = [(f(r[k]), hdr[k][6:]) for k in range(len(hdr)) if hdr[k].startswith("stall_") and "Not Issued" not in hdr[k]]
    stalls.sort(reverse=True)
    res.append((f(r[si]), f(r[ie]), cur_file, r[0], r[1].strip()[:70], stalls[:2]))
tot = sum(x[0] for x in res); toti = sum(x[1] for x in res)
print(f"samples {tot:.0f}  warp-instr {toti:.0f} ({toti / per:.1f} per unit)")
for s, i, fl, ln, src, st in sorted(res, reverse=True)[:top]:
    print(f"{s:6.0f} {100*s/tot:5.1f}% {i/per:8.1f} {fl}:{ln:4s} {src:70s} {st[0][1]}:{st[0][0]:.0f} {st[1][1]}:{st[1][0]:.0f}")
