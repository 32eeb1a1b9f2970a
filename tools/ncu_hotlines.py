"""Top source lines (warp-stall samples) of an ncu report: python tools/ncu_hotlines.py rep [N]."""
import csv, io, subprocess, sys
rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur = None; agg = {}; tot = 0
for r in csv.reader(io.StringIO(out)):
    if len(r) >= 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]; continue
    if len(r) > 8 and r[0] not in ("", "Line No"):
        try:
            s = int(r[4]); ie = int(r[7]); te = int(r[8])
        except ValueError:
            continue
        k = (cur, int(r[0]), r[1][:90]); a = agg.get(k, (0, 0, 0))
        agg[k] = (a[0] + s, a[1] + ie, a[2] + te); tot += s  # summed over launches
print("total samples", tot)
for (f, l, src), (s, ie, te) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:N]:
    print(f"{100*s/max(tot,1):5.1f}% {f}:{l} thr/warp={te/max(ie,1):.1f} | {src}")
