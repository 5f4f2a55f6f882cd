#!/usr/bin/env python
"""Refresh profiles/ from one tools/gpu_check.sh run (plus the other-config / training JSON it leaves):
   python tools/profile_summary.py <tag>      (reads gpurun_out/<tag>/...)
Writes profiles/r01_bench_lowrate.json, r01_launches_lowrate.csv, r01_ncu_final.md, r01_other_configs.jsonl and
the measured header + tables of profiles/r01_summary.md (the hand-written notes below the tables are kept)."""
import json, os, shutil, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1]
src = os.path.join(ROOT, "gpurun_out", tag)
prof = os.path.join(ROOT, "profiles")
shutil.copy(os.path.join(src, "bench.json"), os.path.join(prof, "r01_bench_lowrate.json"))
shutil.copy(os.path.join(src, "launches.csv"), os.path.join(prof, "r01_launches_lowrate.csv"))
if os.path.exists(os.path.join(src, "stages.jsonl")):
    shutil.copy(os.path.join(src, "stages.jsonl"), os.path.join(prof, "r01_other_configs.jsonl"))
run = lambda *a: subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), *a],
                                capture_output=True, text=True).stdout
ncu = run("full", os.path.join(src, "prof_all.ncu-rep"), "lowrate")
open(os.path.join(prof, "r01_ncu_final.md"), "w").write(ncu)
launch = run("launches", os.path.join(prof, "r01_launches_lowrate.csv"))
b = json.load(open(os.path.join(prof, "r01_bench_lowrate.json")))
st, cl, rf = b["stages_ms"], b["clocks"], b["roofline"]
tests = open(os.path.join(src, "pytest.log")).read().strip().splitlines()[-1]
head = f"""# Round 1 — measured path (lowrate: 64×64, M=410, batch 4096, bf16, 1 × B200)

Commands (`tools/gpu_check.sh {tag}`, summarised by `tools/profile_summary.py {tag}`): `python bench.py` (20 timed
steps, 5 warm-up); launch list `ncu --metrics gpu__time_duration.sum --clock-control none python bench.py --steps 2
--warmup 3 --no-cpu-baseline`; full capture `ncu --set full --clock-control none --import-source on -k
regex:"k_conv1_tc|k_conv2_tc|k_conv3_r4|k_proxy" -s 12 -c 4` of the same command. Raw: r01_bench_lowrate.json,
r01_launches_lowrate.csv; per-kernel metrics: r01_ncu_final.md (dram bytes per launch also in traffic.json); other
configs: r01_other_configs.jsonl. GPU tests of the same call: {tests}. (r01_*_tc13.* are an earlier capture of this
round, right after conv layers 1 and 3 moved to the tensor cores; kept for the progression.)

| | start of round | final bench ({tag}) |
|---|---|---|
| step (device, CUDA events) | 20.34 ms | **{b['ms_per_step']:.2f} ms** |
| images/s (device-resident) | 201 k | **{b['value']/1e3:.0f} k** |
| images/s e2e (host y in, host x̂ out) | 189 k | **{b['e2e']['value']/1e3:.0f} k** |
| proxy (Φᵀy, tcgen05) | 0.047 ms | {st['proxy']:.3f} ms (two batch tiles per CTA share each Φᵀ K-block; tile-blocked Φᵀ) |
| conv1 | 5.44 ms (SIMT) | **{st['conv1']:.2f} ms** (tcgen05 .ws, im2row, TMA strip) |
| conv2 | 6.63 ms, 1255 TFLOP/s | **{st['conv2']:.2f} ms, {rf['achieved']:.0f} TFLOP/s = {100*rf['frac']:.0f} % of the measured bf16 burst {rf['peak']:.0f} ({100*rf['frac_of_sustained']:.0f} % of the sustained 1354; {100*rf.get('frac_of_design_ceiling', 0):.0f} % of the tap-stacked form's useful-MAC ceiling {rf.get('design_ceiling', 0):.3f})**; strip pitch 69, weight stream multicast across CTA pairs |
| conv3 | 8.22 ms (SIMT) | **{st['conv3']:.2f} ms** (tcgen05, 8 output rows stacked in M over the resident tap-row stack) |

Clocks during the timed region (NVML in its own process, {cl['samples']} timestamped samples inside the region): median
{cl['sm_mhz']:.0f} MHz under load (max {cl['sm_max_mhz']:.0f}), throttle reasons: {', '.join(cl['reasons']) or 'none'} (kept per the
recipe; the clock is data- and power-dependent, DESIGN.md §11, hence a run-to-run spread of conv2 of about ±3 %
across boxes). CPU baseline (fp64 oracle): {b['cpu_baseline']['value']:.0f} images/s on {b['cpu_baseline']['cores']} host threads;
{b['cpu_baseline']['single_thread_s_per_image']:.2f} s per image on one thread.
"""
old = open(os.path.join(prof, "r01_summary.md")).read()
start = old.index("\nRun-to-run") if "\nRun-to-run" in old else old.index("\nOther configs")
keep = old[start:old.index("## Launch list")]   # hand-written notes between the header and the tables
tail = old[old.index("## Where conv2's issuing thread waits"):]
out = (head + keep + "## Launch list (cold-cache, serialised; compare shares — the e2e part of the command runs chunked "
       "batches, so\n## per-launch means mix batch sizes)\n\n" + launch + f"\n## ncu --set full (one launch each, capture {tag})\n\n"
       + ncu + "\n" + tail)
open(os.path.join(prof, "r01_summary.md"), "w").write(out)
print("profiles refreshed from", tag)
