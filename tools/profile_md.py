"""Assemble profiles/<tag>_bench.md from one tools/gpu_round2.sh <tag> pass:
  python tools/profile_md.py <tag> "<title>" > profiles/<tag>_bench.md
(bench line, the whole-iteration roofline, the serialised launch list and
the ncu --set full summary of the captured kernels)."""
import json
import os
import subprocess
import sys

tag, title = sys.argv[1], sys.argv[2]
out = "gpurun_out"
d = json.load(open(f"{out}/{tag}_bench.json"))
print(f"# {title}\n")
print(f"One B200 (gpurun). `tools/gpu_round2.sh {tag}`: `python bench.py` (no profiler), then the\n"
      "per-launch list of one config-3 iteration (`ncu --metrics gpu__time_duration.sum --clock-control none`,\n"
      "serialised and cold-ish: compare shares, not absolutes) and `ncu --set full` captures of the rollout,\n"
      "head and fused dM + Adam kernels.\n")
print("## Bench line\n\n```json\n" + json.dumps(d) + "\n```\n")
it = d["roofline"]["iteration"]
print("## Whole-iteration roofline (SURVEY §8d, from the bench's per-launch profile pass)\n")
print(f"roofline {it['roofline_ms']} ms vs measured {round(it['measured_ms'], 4)} ms: frac {round(it['frac'], 3)}\n")
print("| phase | GFLOP | GB | ms @ bf16 peak | ms @ HBM peak | bound |\n|---|---|---|---|---|---|")
for k, v in it["phases"].items():
    print(f"| {k} | {v['gflop']} | {v['gbytes']} | {v['ms_tensor']} | {v['ms_hbm']} | {v['bound']} |")
print("\n## Launch list of one config-3 iteration (serialised)\n\n```")
print(subprocess.run([sys.executable, "tools/launchsum.py", f"{out}/{tag}_launches.csv"], capture_output=True,
                     text=True).stdout.rstrip())
print("```\n\n## ncu --set full\n")
raw = f"/tmp/{tag}_raw.csv"
with open(raw, "w") as f:
    subprocess.run(["ncu", "-i", f"{out}/{tag}_prof_misc.ncu-rep", "--page", "raw", "--csv"], stdout=f, check=True)
print(subprocess.run([sys.executable, "tools/ncu_summary.py", raw], capture_output=True, text=True).stdout.rstrip())
os.remove(raw)
