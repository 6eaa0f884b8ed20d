"""Per-opcode instruction mix and warp-stall samples of one kernel launch in an ncu report
(`--set full --import-source on`), normalised per element sorted.

    python tools/sass_mix.py gpurun_out/full_round_H.ncu-rep -k k_classify -s 0 --elems 268435456
"""
import argparse
import collections
import csv
import subprocess


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("-k", "--kernel", required=True)
    ap.add_argument("-s", "--launch", type=int, default=0)
    ap.add_argument("--elems", type=float, required=True, help="elements the launch processed")
    ap.add_argument("--top", type=int, default=20)
    a = ap.parse_args()
    out = subprocess.run(["ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source", "sass",
                          "-k", f"regex:{a.kernel}", "-s", str(a.launch), "-c", "1"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    heads = [i for i, r in enumerate(rows) if r and r[0] == "Address"]
    hdr = rows[heads[0]]
    end = heads[1] - 1 if len(heads) > 1 else len(rows)
    ie, isrc, ist = (hdr.index("Instructions Executed"), hdr.index("Source"),
                     hdr.index("Warp Stall Sampling (All Samples)"))
    ops, stalls = collections.Counter(), collections.Counter()
    tot = tots = 0.0
    for r in rows[heads[0] + 1:end]:
        if len(r) <= ie:
            continue
        try:
            e, s = float(r[ie] or 0), float(r[ist] or 0)
        except ValueError:
            continue
        toks = r[isrc].split()
        if not toks:
            continue
        op = (toks[1] if toks[0].startswith("@") else toks[0]).split(".")[0]
        ops[op] += e
        stalls[op] += s
        tot += e
        tots += s
    print(f"warp instructions {tot:.0f}; thread instructions per element {tot * 32 / a.elems:.1f}")
    print("| opcode | share of instructions | per element | share of stall samples |")
    print("|---|---|---|---|")
    for op, c in ops.most_common(a.top):
        print(f"| {op} | {c / tot:.1%} | {c * 32 / a.elems:.2f} | {stalls[op] / max(tots, 1):.1%} |")


if __name__ == "__main__":
    main()
