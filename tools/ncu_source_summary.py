"""Summarise an ncu report's source page by CUDA source line: warp-stall samples,
executed instructions and the dominant stall reasons (reads `ncu -i X --page source`)."""
import csv
import subprocess
import sys


def main(rep, top=25, kernel=None, launch=0):
    cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"]
    if kernel:
        cmd += ["-k", f"regex:{kernel}", "-s", str(launch), "-c", "1"]
    out = subprocess.run(cmd, capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = None
    fname = ""
    agg = []
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr and r[0].isdigit():
            d = dict(zip(hdr, r))
            try:
                samples = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
                inst = int(d.get("Instructions Executed", "0") or 0)
            except ValueError:
                continue
            stalls = {k[6:]: int(v) for k, v in d.items() if k.startswith("stall_") and "Not Issued" not in k
                      and v.isdigit() and int(v) > 0}
            top3 = sorted(stalls.items(), key=lambda x: -x[1])[:3]
            agg.append((samples, inst, f"{fname}:{r[0]}", r[1].strip()[:70], top3))
    tot_s = sum(a[0] for a in agg) or 1
    tot_i = sum(a[1] for a in agg) or 1
    print(f"total samples {tot_s}, total warp instructions {tot_i}")
    for s, i, loc, src, t3 in sorted(agg, key=lambda x: -x[0])[:top]:
        print(f"{100*s/tot_s:5.1f}% smp {100*i/tot_i:5.1f}% inst  {loc:24s} {src:70s} {t3}")


if __name__ == "__main__":
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--top", type=int, default=25)
    ap.add_argument("-k", "--kernel", default=None)
    ap.add_argument("-s", "--launch", type=int, default=0)
    a = ap.parse_args()
    main(a.rep, a.top, a.kernel, a.launch)
