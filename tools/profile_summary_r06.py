#!/usr/bin/env python
"""Round-2 final evidence summary (r06 captures) from one gpurun capture (tools/scratch/<tag>.sh):
   python tools/profile_summary_r06.py <tag>     (reads gpurun_out/<tag>/, writes profiles/r06_*)
Files: r06_bench_lowrate.json (the bench line), r06_launches_lowrate.csv (+ table), r06_ncu_full.md (per-kernel
--set full metrics; dram bytes per launch also into traffic.json), r06_ncu_pair_stress.md (the lifting GEMM on CTA
pairs at Stress), r06_other_configs.jsonl (per-stage times of the other configs), r06_summary.md (the overview)."""
import json, os, shutil, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1]
src = os.path.join(ROOT, "gpurun_out", tag)
prof = os.path.join(ROOT, "profiles")
cp = lambda a, b: shutil.copy(os.path.join(src, a), os.path.join(prof, b))
cp("bench.json", "r06_bench_lowrate.json")
cp("launches.csv", "r06_launches_lowrate.csv")
cp("stages.jsonl", "r06_other_configs.jsonl")
run = lambda *a: subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), *a],
                                capture_output=True, text=True).stdout
full = run("full", os.path.join(src, "prof_all.ncu-rep"), "lowrate")
open(os.path.join(prof, "r06_ncu_full.md"), "w").write(full)
pair = run("full", os.path.join(src, "prof_pair.ncu-rep"), "stress") if os.path.exists(
    os.path.join(src, "prof_pair.ncu-rep")) else "(no capture)\n"
open(os.path.join(prof, "r06_ncu_pair_stress.md"), "w").write(pair)
launch = run("launches", os.path.join(prof, "r06_launches_lowrate.csv"))
b = json.load(open(os.path.join(prof, "r06_bench_lowrate.json")))
pk_hbm = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6556
st, cl, rf = b["stages_ms"], b["clocks"], b["roofline"]
tests = open(os.path.join(src, "pytest.log")).read().strip().splitlines()[-1]
gpu = open(os.path.join(src, "gpu.txt")).read().strip().replace("\n", "; ")
stages = [json.loads(l) for l in open(os.path.join(src, "stages.jsonl")) if l.startswith("{")]
rows = "\n".join(f"| {s['cfg']} | {s['prec']} | {s['batch']} | {' / '.join(f'{x:.3f}' for x in s['stages_ms'])} | "
                 f"{s['total_ms']:.2f} | {s['images_per_s'] / 1e3:.1f} k | {s['conv2_tflops']:.0f} |" for s in stages)
e2 = b["e2e"]
if "api" in e2:   # streamed headline + blocking
    e2e_rows = (f"| images/s end to end, streamed (`di_recover_host_async` per step, pinned host y in, host x̂ out) | "
                f"**{e2['value'] / 1e3:.0f} k** |\n| images/s end to end, blocking (`di_recover_host` per step) | "
                f"**{e2['blocking']['value'] / 1e3:.0f} k** |")
else:             # bench lines before the streamed API
    e2e_rows = f"| images/s end to end, blocking (`di_recover_host` per step, pinned host y in, host x̂ out) | **{e2['value'] / 1e3:.0f} k** |"
out = f"""# Round 2 (final) — measured path (capture `{tag}`, {gpu})

Commands (`tools/scratch/{tag}.sh`, summarised by `tools/profile_summary_r06.py {tag}`): the `-m gpu` suite
({tests}); `python bench.py` (20 timed steps, 5 warm-up, output check on); `tools/time_stages.py` per config; launch
list `ncu --metrics gpu__time_duration.sum --clock-control none python bench.py --steps 2 --warmup 3
--no-cpu-baseline --no-check --no-train --no-sustained`; full capture `ncu --set full --clock-control none --import-source on -k
regex:"k_conv1_tc|k_conv2_tc|k_conv3_r4|k_proxy" -s 12 -c 4` of the same command (the fourth recovery, full batch);
`ncu --set full -k regex:k_proxy_pair -s 3 -c 1 python tools/time_stages.py stress 3`.

## Bench line (lowrate: 64×64, M = 410, batch 4096, bf16)

| | value |
|---|---|
| step (device, CUDA events) | **{b['ms_per_step']:.2f} ms** |
| images/s device-resident | **{b['value'] / 1e3:.0f} k** |
{e2e_rows}
| images/s sustained (≈ 2 s back to back after the timed region) | **{b.get('sustained', {}).get('images_s', 0) / 1e3:.0f} k** at {b.get('sustained', {}).get('sm_mhz')} MHz, {b.get('sustained', {}).get('power_w_max')} W max, {', '.join(b.get('sustained', {}).get('reasons') or [])} |
| stages (ms) | lifting {st['proxy']:.3f}, conv1 {st['conv1']:.3f}, conv2 {st['conv2']:.3f}, conv3 {st['conv3']:.3f} |
| conv2 | {rf['achieved']:.0f} TFLOP/s = {rf['frac']:.3f} of the measured burst {rf['peak']:.0f}; {rf.get('frac_at_sm_clock', 0):.3f} of {rf.get('peak_at_sm_clock', 0):.0f} TFLOP/s at the sampled SM clock; design ceiling {rf.get('design_ceiling', 0):.3f} |
| clocks (timed region) | median {cl['sm_mhz']:.0f} MHz (max {cl['sm_max_mhz']:.0f}), reasons: {', '.join(cl['reasons']) or 'none'} |
| output check | {json.dumps(b.get('gather_check'))} |
| CPU oracle | {b['cpu_baseline']['value']:.1f} images/s on {b['cpu_baseline']['cores']} threads ({b['cpu_baseline'].get('cpu_model', '?')}) |

## Other configs (tools/time_stages.py, ms per step: lifting / conv1 / conv2 / conv3)

| config | precision | batch | stages ms | step ms | images/s | conv2 TFLOP/s |
|---|---|---|---|---|---|---|
{rows}

## Launch list (cold-cache, serialised; the e2e part of the command runs chunked batches, so compare the largest
## launch of each kernel)

{launch}

## ncu --set full, one full-batch launch per kernel (`r06_ncu_full.md`)

{full}

## Lifting GEMM on CTA pairs at Stress (`r06_ncu_pair_stress.md`)

{pair}
"""
def opt(name):
    p = os.path.join(src, name)
    return open(p).read().strip() if os.path.exists(p) else "(not captured)"
for f in ("hbm_probe.jsonl", "power.json", "e2e.txt"):
    if os.path.exists(os.path.join(src, f)):
        cp(f, "r06_" + f)
tr, thin = b.get("training", {}), b.get("thin_layers", {})
thin_rows = "\n".join(f"| {k} | {v['launch_ms']:.3f} | {v['bytes_per_px']} | {v['achieved_GBs']:.0f} | {v['frac']:.2f} |"
                       for k, v in thin.items())
dbg = open(os.path.join(src, "pytest_debug.log")).read().strip().splitlines()[-1] if os.path.exists(
    os.path.join(src, "pytest_debug.log")) else "(not run)"
out += f"""
## Training step in the bench line (SURVEY.md §8(f) NEXT-2)

{json.dumps(tr)}

## Thin layers against HBM (bench `thin_layers`; both are shared-memory-port bound, see the ncu lines above)

| kernel | ms | algorithmic B/px | GB/s | of {pk_hbm} GB/s |
|---|---|---|---|---|
{thin_rows}

HBM floors on this box (`tools/scratch/hbm_probe.cu`, best of 10; 2.15 GB written / 1.07 GB read):

```
{opt("hbm_probe.jsonl")}
```

## Power (`tools/scratch/power_probe.py`: the recovery back to back for 3 s, nvml every 5 ms)

```
{opt("power.json")}
```

## DI_DEBUG library (bounded barrier waits, device asserts): `-m gpu` suite

{dbg}
"""
open(os.path.join(prof, "r06_summary.md"), "w").write(out)
print("profiles/r06_* refreshed from", tag)
