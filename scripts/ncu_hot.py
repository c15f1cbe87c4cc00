"""Per-instruction stall hot spots of an ncu report (source page, SASS).
usage: python scripts/ncu_hot.py report.ncu-rep [top_n]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
lines = txt.splitlines()
start = [i for i, l in enumerate(lines) if l.startswith('"Address"')][0]
rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
hdr, rows = rows[0], [r for r in rows[1:] if len(r) == len(rows[0])]
ia, isrc = hdr.index("Address"), hdr.index("Source")
iss, iex = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
tot = sum(int(r[iss] or 0) for r in rows)
print(f"{len(rows)} instructions, {tot} samples")
order = sorted(range(len(rows)), key=lambda i: -int(rows[i][iss] or 0))
for i in order[:top]:
    r = rows[i]
    print(f"{i:5d} {100*int(r[iss])/tot:5.1f}% ex={r[iex]:>8s}  {r[isrc].strip()}")
if "--dump" in sys.argv:
    with open(sys.argv[sys.argv.index("--dump") + 1], "w") as f:
        for i, r in enumerate(rows):
            f.write(f"{i:5d} {r[iex]:>8s} {r[iss]:>6s} {r[isrc].strip()}\n")
