"""Per-source-line shared-memory wavefronts (actual / ideal / excessive) of an ncu report."""
import csv
import io
import subprocess
import sys

src = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
h = rows[hi]
ix = {x: i for i, x in enumerate(h)}
out = []
for r in rows[hi + 1:]:
    if len(r) != len(h) or r[2] != "-" or not r[0].isdigit():
        continue
    try:
        wf = float(r[ix["L1 Wavefronts Shared"]] or 0)
        ide = float(r[ix["L1 Wavefronts Shared Ideal"]] or 0)
    except ValueError:
        continue
    if wf > 0:
        out.append((int(wf), int(ide), int(wf - ide), r[0], r[1].strip()[:90]))
out.sort(reverse=True)
print("| wavefronts | ideal | excess | line | source |\n|---|---|---|---|---|")
for o in out[: int(sys.argv[2]) if len(sys.argv) > 2 else 20]:
    print("| %d | %d | %d | %s | `%s` |" % o)
