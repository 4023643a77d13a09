"""Summarise an ncu source page (cuda,sass) by CUDA source line: stall samples
and executed instructions.  usage: python tools/ncu_lines.py rep.ncu-rep [topN]"""
import csv, subprocess, sys, collections
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
samples = collections.Counter(); insts = collections.Counter(); text = {}
cur_file = None; cur_line = None
for row in rows:
    if len(row) == 2 and row[0] == "File Path":
        cur_file = row[1].split("/")[-1]; continue
    if len(row) < 8 or row[0] == "Line No":
        continue
    if row[0]:
        cur_line = (cur_file, int(row[0])); text[cur_line] = row[1].strip()
    try:
        s = float(row[4] or 0); n = float(row[7] or 0)
    except ValueError:
        continue
    if cur_line:
        samples[cur_line] += s; insts[cur_line] += n
tot = sum(samples.values()) or 1; toti = sum(insts.values()) or 1
print(f"total stall samples {tot:.0f}, executed warp instructions {toti:.0f}")
for k, s in samples.most_common(top):
    print(f"{100*s/tot:5.1f}% samp {100*insts[k]/toti:5.1f}% inst  {k[0]}:{k[1]:<5d} {text.get(k,'')[:90]}")
