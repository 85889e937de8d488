"""Per-source-line instruction and stall shares of an .ncu-rep in SOURCE order (lines above a threshold):
python tools/ncu_src.py <rep> [min_pct]"""
import csv, subprocess, sys

def main(path, thr=0.4):
    txt = subprocess.run(["ncu", "-i", path, "--page", "source", "--print-source", "cuda,sass", "--csv"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    hdr = next(r for r in rows if r and r[0] == "Line No")
    ii, st = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
    fname, lines = "", []
    for r in rows:
        if r and r[0] == "File Path":
            fname = r[1].split("/")[-1]
        elif len(r) > ii and r[0].isdigit() and r[ii].isdigit():
            lines.append((int(r[ii]), int(r[st]) if r[st].isdigit() else 0, fname, int(r[0]), r[1].strip()))
    tot, tots = sum(l[0] for l in lines) or 1, sum(l[1] for l in lines) or 1
    print(f"# {path}: {tot} warp instructions, {tots} stall samples")
    for n, s, f, ln, src in sorted(lines, key=lambda x: (x[2], x[3])):
        if 100 * n / tot >= thr or 100 * s / tots >= thr:
            print(f"{100 * n / tot:5.1f}% inst {100 * s / tots:5.1f}% stall  {f}:{ln}: {src[:100]}")

if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else 0.4)
