"""Per-region view of an ncu report's SASS page: executed instructions and stall
samples per stretch between markers (BAR.SYNC, loop back-edges), plus the hottest lines.

    python tools/sass_profile.py gpurun_out/prof_x.ncu-rep [top]
"""
import csv
import io
import subprocess
import sys


def load(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    lines = out.splitlines()
    rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
    hdr = rows[0]
    return hdr, rows[1:]


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    hdr, rows = load(path)
    ia = hdr.index("Address")
    isrc = hdr.index("Source")
    iex = hdr.index("Instructions Executed")
    ism = hdr.index("Warp Stall Sampling (All Samples)")
    iwf = hdr.index("L1 Wavefronts Shared") if "L1 Wavefronts Shared" in hdr else None
    iwi = hdr.index("L1 Wavefronts Shared Ideal") if "L1 Wavefronts Shared Ideal" in hdr else None

    def num(v):
        try:
            return float(v.replace(",", ""))
        except ValueError:
            return 0.0
    tot_ex = sum(num(r[iex]) for r in rows)
    tot_sm = sum(num(r[ism]) for r in rows)
    print(f"total warp instructions {tot_ex:.4g}, stall samples {tot_sm:.4g}")
    # regions split at barriers
    reg, ex, sm, wf, wfi, start = 0, 0.0, 0.0, 0.0, 0.0, rows[0][ia]
    for r in rows:
        ex += num(r[iex])
        sm += num(r[ism])
        if iwf is not None:
            wf += num(r[iwf])
            wfi += num(r[iwi])
        if "BAR.SYNC" in r[isrc] or r is rows[-1]:
            print(f"region {reg:2d} [{start}..{r[ia]}]: {ex / tot_ex:6.1%} of instructions, "
                  f"{sm / max(tot_sm, 1):6.1%} of stall samples, smem wavefronts {wf:.3g} (ideal {wfi:.3g})")
            reg += 1
            ex = sm = wf = wfi = 0.0
            start = r[ia]
    print("hottest instructions by stall samples:")
    for r in sorted(rows, key=lambda r: -num(r[ism]))[:top]:
        print(f"  {r[ia]} {num(r[ism]) / max(tot_sm, 1):6.2%} ex={num(r[iex]):.3g}  {r[isrc][:90]}")


if __name__ == "__main__":
    main()
