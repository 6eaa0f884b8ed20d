"""Per CUDA source line: shared-memory wavefronts (actual / ideal) and instructions, from an
ncu report's source page (tools only)."""
import csv
import subprocess
import sys
from collections import defaultdict


def main(rep, kernel, launch=0, top=25):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                          "-k", f"regex:{kernel}", "-s", str(launch), "-c", "1"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = None
    agg = defaultdict(lambda: [0, 0, 0, ""])
    cur = None
    for r in rows:
        if not r:
            continue
        if r[0] == "Line No" and len(r) > 10:
            hdr = r
            continue
        if hdr and r[0].isdigit():
            d = dict(zip(hdr, r))
            src = r[1].strip()
            key = (int(r[0]), src[:90])
            def num(x):
                try:
                    return int(float(x or 0))
                except ValueError:
                    return 0
            a = agg[key]
            a[0] += num(d.get("L1 Wavefronts Shared"))
            a[1] += num(d.get("L1 Wavefronts Shared Ideal"))
            a[2] += num(d.get("Instructions Executed"))
    tot = sum(v[0] for v in agg.values()) or 1
    toti = sum(v[2] for v in agg.values()) or 1
    print(f"total shared wavefronts {tot}, warp instructions {toti}")
    for (ln, src), (wf, ideal, ins, _) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{100*wf/tot:5.1f}% wf (ideal {ideal/max(wf,1):4.2f})  {100*ins/toti:5.1f}% inst  {ln:5d} {src}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 0)
