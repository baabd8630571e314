#!/usr/bin/env python
"""Turn a gpu_evidence.sh run (gpurun_out/ev/) into the committed profiles/:
bench JSON lines, launch-list summaries, ncu --set full summaries of K2 per
config, and profiles/traffic.json (DRAM bytes per K2 launch, read by bench.py).

    python scripts/make_profiles.py r01
"""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EV = os.path.join(ROOT, "gpurun_out", "ev")
OUT = os.path.join(ROOT, "profiles")
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_shared_mem", "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum",
        "sm__cycles_elapsed.avg.per_second"]
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def ncu_raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    return r[0], r[1], r[2]


def summarize_ncu(rep, cfg, tag, kern="k_tasks", skip=3):
    h, u, v = ncu_raw(rep)
    get = lambda k: (v[h.index(k)], u[h.index(k)]) if k in h else (None, None)
    lines = [f"# ncu --set full: K2 (k_tasks), config C{cfg} ({tag})", "",
             f"kernel: `{v[h.index('Kernel Name')][:140]}`", "",
             f"command: `ncu --set full --clock-control none --import-source on -k regex:{kern} -s {skip} -c 1 "
             f"python bench.py --config {cfg} --steps 3 --warmup 3 --no-extras`", "",
             "| metric | value | unit |", "|---|---|---|"]
    for k in KEYS:
        val, un = get(k)
        if val is not None:
            lines.append(f"| {k} | {val} | {un} |")
    st = []
    for i, k in enumerate(h):
        if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
            try:
                st.append((float(v[i]), k[len("smsp__pcsamp_warps_issue_stalled_"):]))
            except ValueError:
                pass
    tot = sum(s for s, _ in st) or 1
    lines += ["", "warp-stall samples: " + ", ".join(f"{n} {s / tot * 100:.0f}%" for s, n in sorted(st, reverse=True)[:8])]
    rd, ur = get("dram__bytes_read.sum")
    wr, uw = get("dram__bytes_write.sum")
    traffic = float(rd) * UNIT.get(ur, 1) + float(wr) * UNIT.get(uw, 1)
    dur, ud = get("gpu__time_duration.sum")
    return "\n".join(lines) + "\n", traffic, float(dur) * (1e-3 if ud == "us" else (1.0 if ud == "ms" else 1e-6))


def summarize_launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10 and r[0] != "ID"]
    agg = {}
    for r in rows:
        name = r[4].split("(")[0].replace("void ", "")[:70]
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += float(r[-1])
    ours = sum(v[1] for k, v in agg.items() if k.startswith("sm::"))
    lines = ["| kernel | launches | total us | avg us | share of library time |", "|---|---|---|---|---|"]
    for k, v in agg.items():
        share = f"{v[1] / ours:.3f}" if k.startswith("sm::") and ours else "-"
        lines.append(f"| `{k}` | {v[0]} | {v[1] / 1e3:.1f} | {v[1] / v[0] / 1e3:.2f} | {share} |")
    return "\n".join(lines) + "\n"


def main(tag):
    os.makedirs(OUT, exist_ok=True)
    traffic = {}
    rows = []
    for cfg in (2, 1, 3, 4, 5, 6):
        blog = os.path.join(EV, "bench_default.log" if cfg == 2 else f"bench_c{cfg}.log")
        line = None
        if os.path.exists(blog):
            for ln in open(blog):
                if ln.startswith("{"):
                    line = json.loads(ln)
        if line:
            json.dump(line, open(os.path.join(OUT, f"{tag}_bench_c{cfg}.json"), "w"))
        rep = os.path.join(EV, f"{tag}_c{cfg}_k_tasks.ncu-rep")
        tr = None
        if os.path.exists(rep):
            text, tr, dur = summarize_ncu(rep, cfg, tag)
            open(os.path.join(OUT, f"{tag}_ncu_k_tasks_c{cfg}.md"), "w").write(text)
            traffic[str(cfg)] = {"dram_bytes_per_launch": tr, "ncu_duration_ms": dur,
                                 "source": f"profiles/{tag}_ncu_k_tasks_c{cfg}.md (dram__bytes_read.sum + "
                                           "dram__bytes_write.sum, one ncu --set full capture)"}
        lpath = os.path.join(EV, f"{tag}_launches_c{cfg}.csv")
        if os.path.exists(lpath):
            open(os.path.join(OUT, f"{tag}_launches_c{cfg}.md"), "w").write(
                f"# ncu launch list, config C{cfg} ({tag})\n\n`ncu --metrics gpu__time_duration.sum --clock-control "
                f"none python bench.py --config {cfg} --steps 3 --warmup 3 --no-extras` -- cold-cache, serialised "
                f"per-launch times: compare shares, not absolutes\n\n" + summarize_launches(lpath))
        if line:
            rf = line.get("roofline", {})
            rows.append((cfg, line, rf, tr))
    # extra captures: K1 on C2, K3 on C5; the merge-path comparison line
    for name, rep in (("k_cross_ranks_c2", f"{tag}_c2_k_cross_ranks"), ("k_block_sort_c5", f"{tag}_c5_k_block_sort")):
        path = os.path.join(EV, rep + ".ncu-rep")
        if os.path.exists(path):
            kern = name.split("_c")[0]
            text, tr, dur = summarize_ncu(path, 2 if "c2" in name else 5, tag, kern, 3 if "c2" in name else 1)
            text = text.replace("K2 (k_tasks)", name.split("_c")[0])
            open(os.path.join(OUT, f"{tag}_ncu_{name}.md"), "w").write(text)
    mp = os.path.join(EV, "bench_c2_mergepath.log")
    if os.path.exists(mp):
        for ln in open(mp):
            if ln.startswith("{"):
                json.dump(json.loads(ln), open(os.path.join(OUT, f"{tag}_bench_c2_mergepath.json"), "w"))
    ref = os.path.join(EV, "bench_reference.log")
    if os.path.exists(ref):
        for ln in open(ref):
            if ln.startswith("{"):
                json.dump(json.loads(ln), open(os.path.join(OUT, f"{tag}_bench_reference.json"), "w"))
    pt = os.path.join(EV, "pytest_gpu.log")
    if os.path.exists(pt):
        open(os.path.join(OUT, f"{tag}_pytest_gpu.log"), "w").write(open(pt).read())
    json.dump(traffic, open(os.path.join(OUT, "traffic.json"), "w"), indent=1)
    print(json.dumps(traffic, indent=1))
    write_readme(tag, rows, traffic)
    for cfg, line, rf, tr in rows:
        print(cfg, f"{line['value']:.4g} elem/s", f"{line['ms_per_step']:.4f} ms", f"{line.get('achieved_hbm_gbs', 0):.0f} GB/s",
              f"K2 {rf.get('achieved', 0):.0f} GB/s frac {rf.get('frac', 0):.3f}", "traffic", tr,
              "alg", rf.get("algorithmic_bytes_per_launch"))


NAMES = {1: "C1 merge 2^20+2^20 u32+u32", 2: "C2 merge 2^26+2^26 i32 keys-only (default)",
         3: "C3 merge 2^28+2^16 i64+u32", 4: "C4 merge 2^27+2^25 u64+u32", 5: "C5 sort 2^28 u32+u32",
         6: "B1 batched 2^16 pairs u32+u32 (NEXT row)"}


def write_readme(tag, rows, traffic):
    out = [f"# Profiles and measurements -- {tag}", "",
           "One B200 (gpurun, `scripts/gpu_evidence.sh`, then `scripts/make_profiles.py`).  Peak = "
           "MEASURED_PEAKS.json `hbm_gbs` (measured copy, read+write); every `frac` is of that measured peak.  "
           "Clocks: NVML samples inside each timed region (in each bench line); no throttle reason other than "
           "`sw_power_cap` is accepted.", "",
           "| Config | ms/step | elements/s | step GB/s (frac) | K2 GB/s (frac) | K2 share | K2 DRAM traffic / algorithmic "
           "| e2e elements/s (host buffers) | CPU oracle elements/s (1 core) | clocks |",
           "|---|---|---|---|---|---|---|---|---|---|"]
    for cfg, line, rf, tr in rows:
        clk = line.get("clocks", {})
        out.append(f"| {NAMES.get(cfg, cfg)} | {line['ms_per_step']:.4f} | {line['value']:.3e} | "
                   f"{line['achieved_hbm_gbs']:.0f} ({line['achieved_hbm_frac']:.3f}) | {rf.get('achieved', 0):.0f} "
                   f"({rf.get('frac', 0):.3f}) | {rf.get('share_of_step', 0):.3f} | "
                   f"{(tr / rf['algorithmic_bytes_per_launch']) if tr else float('nan'):.3f} | "
                   f"{line.get('e2e', {}).get('value', float('nan')):.3e} | "
                   f"{line.get('cpu_baseline', {}).get('value', float('nan')):.3e} | "
                   f"{clk.get('sm_mhz')} MHz {clk.get('reasons')} |")
    mp = os.path.join(OUT, f"{tag}_bench_c2_mergepath.json")
    if os.path.exists(mp):
        d = json.load(open(mp))
        out += ["", f"Merge-path comparison (not the method; `bench.py --merge-path`, C2): {d['ms_per_step']:.4f} "
                    f"ms/step, {d['value']:.3e} elements/s, {d['achieved_hbm_gbs']:.0f} GB/s "
                    f"({d['achieved_hbm_frac']:.3f}) -- see DESIGN.md for what it measures."]
    out += ["", "Files:",
            f"- `{tag}_bench_cN.json` -- the bench.py JSON line of config N (default N=2).",
            f"- `{tag}_launches_cN.md` -- ncu launch list of `bench.py --config N --steps 3 --warmup 3 --no-extras` "
            "(`--metrics gpu__time_duration.sum --clock-control none`): per-kernel share of the library's time.",
            f"- `{tag}_ncu_k_tasks_cN.md` -- one `ncu --set full` capture of K2 per config (DRAM bytes, throughput, "
            "shared-memory pipe, bank conflicts, occupancy, issue, warp stalls); "
            f"`{tag}_ncu_k_cross_ranks_c2.md` (K1) and `{tag}_ncu_k_block_sort_c5.md` (K3).",
            "- `traffic.json` -- DRAM read+write bytes per K2 launch from those captures (bench.py `roofline.traffic`).",
            f"- `{tag}_bench_reference.json` -- `bench.py --impl reference`: the CPU oracle as the reference arm.",
            "- `r01_size_sweep.md` -- merge throughput against size (`scripts/size_sweep.sh`, round 1, written by hand).",
            f"- `{tag}_pytest_gpu.log` -- the full `pytest -m gpu` run on the B200."]
    open(os.path.join(OUT, "README.md"), "w").write("\n".join(out) + "\n")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r01")
