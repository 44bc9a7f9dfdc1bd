"""Top SASS lines by executed instructions / stall samples from an ncu report:
  python tools/ncu_hot.py gpurun_out/x.ncu-rep [kernel-regex] [N]"""
import csv, io, subprocess, sys

rep = sys.argv[1]
k = sys.argv[2] if len(sys.argv) > 2 else None
N = int(sys.argv[3]) if len(sys.argv) > 3 else 40
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"]
if k:
    cmd += ["-k", "regex:" + k]
out = subprocess.run(cmd, capture_output=True, text=True).stdout
lines = out.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
end = next((i for i in range(start + 1, len(lines)) if lines[i].startswith('"Kernel Name"')), len(lines))
rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:end]))))  # first kernel instance
tot = sum(float(r["Instructions Executed"] or 0) for r in rows)
samp = sum(float(r["Warp Stall Sampling (All Samples)"] or 0) for r in rows)
print(f"total inst {tot:.0f}  samples {samp:.0f}  sass lines {len(rows)}")
rows.sort(key=lambda r: -float(r["Instructions Executed"] or 0))
for i, r in enumerate(rows[:N]):
    print(f'{i:3d} {r["Address"][-5:]} inst {float(r["Instructions Executed"]):9.0f} samp {r["Warp Stall Sampling (All Samples)"]:>5}  {r["Source"].strip()[:70]}')
