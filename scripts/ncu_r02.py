"""Summarise the ncu captures of scripts/prof_r02.sh ON THE GPU BOX (the .ncu-rep files are too
large to bring back): per capture, gpurun_out/ncu_<name>.json with the fields bench.py reads
(kernel_mangled, dram bytes per path*term or per path*window) plus the occupancy / pipe / stall /
opcode / shared-memory figures, and the source page (per-SASS-line stalls) as a gzipped CSV.

usage: python scripts/ncu_r02.py name ...   (then rm gpurun_out/prof_*.ncu-rep)
"""
import csv
import gzip
import hashlib
import io
import json
import os
import subprocess
import sys
from collections import Counter

OUT = "gpurun_out"
UNIT = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "msecond": 1e-3, "usecond": 1e-6, "nsecond": 1e-9,
        "second": 1.0, "ms": 1e-3, "us": 1e-6, "ns": 1e-9, "s": 1.0, "GB": 1e9, "MB": 1e6, "KB": 1e3, "B": 1.0}


def raw(rep, mangled=False):
    cmd = ["ncu", "-i", rep, "--page", "raw", "--csv"] + (["--print-kernel-base", "mangled"] if mangled else [])
    r = list(csv.reader(io.StringIO(subprocess.run(cmd, capture_output=True, text=True).stdout)))
    return {h: (v, u) for h, u, v in zip(r[0], r[1], r[2])}


def main():
    for name in sys.argv[1:]:
        rep = os.path.join(OUT, f"prof_{name}.ncu-rep")
        if not os.path.exists(rep):
            print(name, "no report")
            continue
        d = raw(rep)
        dm = raw(rep, mangled=True)

        def f(k):
            try:
                v, u = d[k]
                return float(v) * UNIT.get(u, 1.0)
            except Exception:
                return None
        with open(os.path.join(OUT, f"plain_{name}.log")) as fh:
            line = json.loads([x for x in fh if x.startswith("{")][-1])
        roof = line["roofline"]
        paths = line["config"]["paths_per_gpu"]
        n = line["config"]["grid"] ** 2
        spk = line.get("path_terms_per_window")
        hyb = roof.get("hybrid_paths") or 0
        traffic = f("dram__bytes_read.sum") + f("dram__bytes_write.sum")
        dur = f("gpu__time_duration.sum")
        stream = name.startswith(("tma", "var", "xs"))
        live = (hyb if "_hybrid" in name else paths)
        stalls = {k[34:-23]: float(v[0]) for k, v in d.items()
                  if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")}
        src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                             capture_output=True, text=True).stdout
        with gzip.open(os.path.join(OUT, f"src_{name}.csv.gz"), "wt") as fh:
            fh.write(src)
        mix = Counter()
        try:
            rows = list(csv.reader(io.StringIO(src)))
            h = rows[1]
            ia, isrc = h.index("Instructions Executed"), h.index("Source")
            for x in rows[2:]:
                toks = x[isrc].split()
                if toks:
                    mix[(toks[1] if toks[0].startswith("@") else toks[0]).split(".")[0]] += float(x[ia] or 0)
        except Exception:
            pass
        tot = sum(mix.values()) or 1.0
        lib = os.path.join("paper_2207_09776_b200", "lib", "libspde2d_b200.so")
        sys.path.insert(0, os.getcwd())
        from bench import sass_sha256
        s = {
            "kernel": d["Kernel Name"][0],
            "lib_sha256": hashlib.sha256(open(lib, "rb").read()).hexdigest(),
            "kernel_mangled": dm["Kernel Name"][0],
            "sass_sha256": sass_sha256(dm["Kernel Name"][0]),
            "capture": f"ncu --set full --clock-control none --import-source on, one launch; scripts/prof_r02.sh {name}",
            "duration_ms": dur * 1e3,
            "dram_bytes_read": f("dram__bytes_read.sum"),
            "dram_bytes_write": f("dram__bytes_write.sum"),
            "dram_bytes_total": traffic,
            "achieved_dram_GBps": traffic / dur / 1e9,
            "registers_per_thread": f("launch__registers_per_thread"),
            "grid_ctas": f("launch__grid_size"),
            "block_threads": f("launch__block_size"),
            "shared_bytes_per_cta": f("launch__shared_mem_per_block_dynamic"),
            "warps_active_pct": f("sm__warps_active.avg.pct_of_peak_sustained_active"),
            "issue_active_pct": f("smsp__issue_active.avg.pct_of_peak_sustained_active"),
            "fp64_pipe_pct_of_active": f("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
            "fp64_pipe_pct_of_elapsed": f("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed"),
            "sm_active_over_elapsed": (f("sm__cycles_active.avg") or 0) / (f("sm__cycles_elapsed.avg") or 1),
            "shared_wavefronts": f("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"),
            "shared_bank_conflicts": f("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"),
            "shared_pipe_pct": f("l1tex__data_pipe_lsu_wavefronts_mem_shared.avg.pct_of_peak_sustained_elapsed"),
            "l2_hit_pct": f("lts__t_sector_hit_rate.pct"),
            "instructions": f("smsp__inst_executed.sum"),
            "top_stalls_cycles_per_issue": dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:10]),
            "opcode_mix_pct": {k: round(v / tot * 100, 2) for k, v in mix.most_common(14)},
            "bench_line": {"config": line["config"]["workload"], "path_terms_per_window": spk, "hybrid_paths": hyb},
        }
        if name.startswith("em_"):
            # E-M: the cluster kernel runs every step of the timed solve in its launch, em_tb two
            steps = 2 if "em_tb" in s["kernel"] else line["euler_maruyama"]["steps"]
            s["em_steps_in_launch"] = steps
            s["dram_bytes_per_path_step"] = traffic / (paths * steps)
            s["algorithmic_bytes"] = 16.0 * n * paths * steps
            s["traffic_over_algorithmic"] = traffic / s["algorithmic_bytes"]
        elif stream:
            # term_xs2_kernel applies two Taylor terms per launch: 40 B per two terms by design
            tpl = 2 if name.startswith("xs2") else 1
            s["live_paths_in_pass"] = live
            s["terms_per_launch"] = tpl
            s["dram_bytes_per_path_term"] = traffic / live / tpl
            s["algorithmic_bytes"] = (40.0 if tpl == 2 else 32.0) * n * live
            s["traffic_over_algorithmic"] = traffic / s["algorithmic_bytes"]
        else:
            cl = paths - hyb
            s["cluster_paths"] = cl
            s["dram_bytes_per_path_window"] = traffic / cl
            s["algorithmic_bytes_streaming_model"] = 32.0 * n * spk * cl
            s["traffic_over_algorithmic"] = traffic / s["algorithmic_bytes_streaming_model"]
        with open(os.path.join(OUT, f"ncu_{name}.json"), "w") as fh:
            json.dump(s, fh, indent=1)
        print(name, json.dumps({k: s[k] for k in ("duration_ms", "warps_active_pct", "issue_active_pct",
                                                  "fp64_pipe_pct_of_active", "traffic_over_algorithmic")}))


if __name__ == "__main__":
    main()
