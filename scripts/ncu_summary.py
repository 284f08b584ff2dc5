"""Summaries of the ncu captures kept under profiles/ (run here, on the pulled files).

  python scripts/ncu_summary.py launches gpurun_out/launches.csv profiles/r02/ncu_launches_cfg5.txt profiles/ncu_traffic.json cfg5 "<command>"
      ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv
      launch list -> the last local step's launches (split_tokens_k .. the step's last
      adamw_k), per-launch time / share / DRAM bytes, and (merged into the json under the
      configuration's name) the expert-GEMM DRAM bytes per launch that bench.py reports as
      roofline.traffic
  python scripts/ncu_summary.py full gpurun_out/prof.ncu-rep profiles/r01/ncu_full_top_kernels.txt
      ncu --set full capture -> the headline metrics of each captured launch
"""
import csv
import io
import json
import subprocess
import sys


def _rows(text):
    lines = [ln for ln in text.splitlines() if ln.startswith('"')]
    return list(csv.DictReader(io.StringIO("\n".join(lines))))


def launches(csv_path, out_txt, out_json, cfg_name, cmd):
    rows = _rows(open(csv_path).read())
    by_id = {}
    for r in rows:
        e = by_id.setdefault(int(r["ID"]), {"name": r["Kernel Name"], "grid": r["Grid Size"]})
        v = float(r["Metric Value"].replace(",", ""))
        unit = r["Metric Unit"]
        if r["Metric Name"] == "gpu__time_duration.sum":
            e["us"] = v * {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3,
                           "msecond": 1e3}[unit]
        else:
            scale = {"byte": 1, "B": 1, "Kbyte": 1e3, "KB": 1e3, "Mbyte": 1e6, "MB": 1e6,
                     "Gbyte": 1e9, "GB": 1e9}[unit]
            e[r["Metric Name"]] = v * scale
    seq = [by_id[i] for i in sorted(by_id)]
    # a step starts with the token split (layer 0 reads the embedding in place) or the
    # embedding gather
    starts = [i for i, e in enumerate(seq)
              if "split_tokens_k" in e["name"] or "embed_gather_k" in e["name"]]
    if not starts:
        sys.exit("no split_tokens_k / embed_gather_k launch in the list")
    s0 = starts[-1]
    ends = [i for i in range(s0, len(seq)) if "adamw_k" in seq[i]["name"]]
    step = seq[s0:ends[-1] + 1] if ends else seq[s0:]
    total = sum(e["us"] for e in step)
    out = [
        f"# One SPES local step ({cfg_name}, N=1), ncu launch list: gpu__time_duration.sum per launch,",
        "# --clock-control none, serialized and cold-cache (share of the step is what matters;",
        "# in the graph-replayed step the side-stream launches overlap the main stream).",
        f"# Command: {cmd}",
        f"# launches in the step: {len(step)}; sum of kernel durations: {total:.1f} us",
        "      us  share DRAM rd MB DRAM wr MB  kernel",
    ]
    for e in step:
        out.append("%8.1f %5.1f%% %10.1f %10.1f  %s" % (
            e["us"], 100 * e["us"] / total, e.get("dram__bytes_read.sum", 0) / 1e6,
            e.get("dram__bytes_write.sum", 0) / 1e6, e["name"][:110]))
    open(out_txt, "w").write("\n".join(out) + "\n")
    # the six expert contractions: every grouped GEMM of the step except the head's (the
    # forward with the CE epilogue, and the two backward GEMMs between it and combine_bwd)
    head = set()
    hf = [i for i, e in enumerate(step) if "EpiHeadCE" in e["name"] or "head" in e["name"]]
    cb = [i for i, e in enumerate(step) if "combine_bwd_k" in e["name"]]
    if hf and cb:
        head = set(range(hf[0], cb[0]))
    # ... and the router weight-gradient GEMM (the first grouped GEMM after each
    # norm_router_finish_k, above 16 experts)
    for i, e in enumerate(step):
        if "norm_router_finish_k" in e["name"]:
            j = next((j for j in range(i + 1, len(step)) if "grouped_gemm" in step[j]["name"]), None)
            if j is not None and "EpiStoreF32<128>, 1, 1" in step[j]["name"]:
                head.add(j)
    gem = [e for i, e in enumerate(step) if "grouped_gemm" in e["name"] and i not in head]
    summary = {
        "source": f"{out_txt} ({cmd})",
        "kernels": [e["name"][:80] for e in gem],
        "launches_per_step": len(gem),
        "dram_bytes_per_step": sum(e.get("dram__bytes_read.sum", 0) + e.get("dram__bytes_write.sum", 0)
                                   for e in gem),
        "ncu_us_per_step": sum(e["us"] for e in gem),
    }
    summary["gemm_dram_bytes_per_launch"] = summary["dram_bytes_per_step"] / max(1, len(gem))
    try:
        allc = json.load(open(out_json))
    except Exception:
        allc = {}
    allc[cfg_name] = summary
    json.dump(allc, open(out_json, "w"), indent=1)
    print(f"{len(step)} launches, {total:.1f} us; {len(gem)} grouped GEMM launches")


FULL_METRICS = [
    "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
    "launch__block_size", "launch__grid_size", "launch__registers_per_thread",
    "lts__t_sector_hit_rate.pct", "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__m_xbar2l1tex_read_bytes.sum",
]


def full(rep, out_txt, cmd):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    lines = [ln for ln in raw.splitlines() if ln.startswith('"')]
    rd = list(csv.reader(io.StringIO("\n".join(lines))))
    hdr, units, data = rd[0], rd[1], rd[2:]
    out = ["# ncu --set full --clock-control none, one launch each of the captured kernels.",
           f"# Command: {cmd}",
           "# traffic = dram__bytes_read.sum + dram__bytes_write.sum for that launch.", ""]
    for row in data:
        d = dict(zip(hdr, row))
        u = dict(zip(hdr, units))
        out.append(d["Kernel Name"][:120])
        tb = 0.0
        for m in FULL_METRICS:
            if m in d:
                out.append("   %-64s %14s %s" % (m, d[m], u.get(m, "")))
                if m.startswith("dram__bytes"):
                    unit = u.get(m, "Mbyte").strip().strip('"')
                    tb += float(d[m].replace(",", "")) * {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1,
                                                          "Gbyte": 1e3}.get(unit, 1)
        out.append("   traffic_MB %.1f" % tb)
        out.append("")
    open(out_txt, "w").write("\n".join(out) + "\n")
    print(f"{len(data)} launches summarised")


if __name__ == "__main__":
    what = sys.argv[1]
    if what == "launches":
        launches(sys.argv[2], sys.argv[3], sys.argv[4], sys.argv[5],
                 sys.argv[6] if len(sys.argv) > 6 else "")
    elif what == "full":
        full(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else "")
    else:
        sys.exit(__doc__)
