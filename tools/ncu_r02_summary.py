"""Summarise the round-2 per-kernel ncu captures (tools/r02_ncu_all.sh ->
gpurun_out/ncu/*_raw.csv) into profiles/r02_ncu_kernels.json: per launch the
device time, DRAM bytes (ncu), the ALGORITHMIC bytes of the launch (the
compulsory traffic of its work unit, stated per kernel below), achieved
algorithmic GB/s and its fraction of the measured HBM peak, FP64 pipe / issue
activity, occupancy and the top stall reasons.  ncu replays each kernel with
cold caches and serialised launches: the absolute times are pessimistic."""
import csv
import gzip
import json
import shutil
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
SRC = Path(sys.argv[1] if len(sys.argv) > 1 else ROOT / "gpurun_out" / "ncu")
PEAK = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()).get("hbm_gbs", 6551.0) \
    if (ROOT / "MEASURED_PEAKS.json").exists() else 6551.0

MB = 1e6


def algorithmic(cap, name):
    """Compulsory bytes of one launch (see the module doc)."""
    ks2 = ", 2," in name or "2, 1, 2>" in name or ", 2, 0," in name or ", 2, 1>" in name
    if cap in ("kh2d", "kh2d_pair"):   # KH2D 1024^2, 4 comps: r u^s + w out (+ r u^n)
        stage = 2 if (", 1, 0" in name and "pair" in name) or ", 64, 1, 0" in name else 3
        return 1024 * 1024 * 4 * 8 * stage, f"1024^2 cells x 4 comps x 8 B x {stage} (r u^s, w out{', r u^n' if stage == 3 else ''})"
    if cap == "mc_pair" and "pair_kernel" in name:   # batched MC: 16 KH2D instances x 512^2
        stage = 2 if "0, 1, 1, 1, 0>" in name else 3
        return 16 * 512 * 512 * 4 * 8 * stage, f"16 x 512^2 cells x 4 comps x 8 B x {stage}"
    if cap == "mc_pair" and "init_eval" in name:
        return 16 * 512 * 512 * 4 * 8, "16 samples x 512^2 cells x 4 comps x 8 B written"
    if cap == "bqmc_pair":             # 4 Burgers instances x 2048^2, pair kernel (fast default)
        stage = 2 if "1, 0, 1, 1, 0>" in name else 3
        return 4 * 2048 * 2048 * 8 * stage, f"4 x 2048^2 cells x 8 B x {stage}"
    if cap == "bqmc_ring":             # 4 Burgers instances x 2048^2
        stage = 3 if "2, 1, 2>" in name else 2
        return 4 * 2048 * 2048 * 8 * stage, f"4 x 2048^2 cells x 8 B x {stage}"
    if cap == "kh3d":                  # 512^3 x 5 comps
        stage = 2 if "<0, 1, 1, 0>" in name and False else None
        return None, "see ring3 note"
    if "moments_push" in name:
        if cap == "mc_moments":   # batched push: 16 samples read, (mean, M2) read + written once
            return 16 * 512 * 512 * 4 * 8 + 512 * 512 * 4 * 32, \
                "16 samples x 512^2 cells x 4 comps x 8 B read + (mean, M2) rmw 32 B once per batch"
        if cap == "bqmc_stats":
            return 2048 * 2048 * 40, "2048^2 cells x (r u 8 + rmw mean 16 + rmw M2 16) B"
        return 512 * 512 * 4 * 40, "512^2 cells x 4 comps x (r u 8 + rmw mean 16 + rmw M2 16) B"
    if "structure_pass1" in name:
        return 2048 * 2048 * 8, "2048^2 cells x 8 B (one field read; the (H+1) x dim shifted passes hit L2)"
    if "structure_pass2" in name:
        return None, "one block, (H+1) x dim x nblocks partials (latency)"
    if "init_eval" in name:
        return 16 * 512 * 512 * 4 * 8, "16 samples x 512^2 cells x 4 comps x 8 B written"
    if "halo_instances" in name:
        return 4 * 4 * 512 * 2 * 4 * 8 * 2, "4 subdomains x 4 faces x 512 x g=2 x 4 comps x 8 B, read + write"
    return None, ""


def stalls(h, r):
    out = []
    for i, k in enumerate(h):
        if "average_warps_issue_stalled" in k and k.endswith("per_issue_active.ratio"):
            try:
                v = float(r[i])
            except ValueError:
                continue
            if v > 0.1:
                out.append((k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""),
                            round(v, 2)))
    return dict(sorted(out, key=lambda kv: -kv[1])[:6])


def val(h, r, k, scale=1.0):
    try:
        return float(r[h.index(k)].replace(",", "")) * scale
    except (ValueError, IndexError):
        return None


def main():
    res = []
    dest = ROOT / "profiles" / "r02_ncu"
    dest.mkdir(parents=True, exist_ok=True)
    for f in sorted(SRC.glob("*_raw.csv")):
        cap = f.name[:-len("_raw.csv")]
        rows = list(csv.reader(open(f)))
        if len(rows) < 3:
            continue
        h, units = rows[0], rows[1]
        unit = {k: units[i] for i, k in enumerate(h)}
        for idx, r in enumerate(rows[2:]):
            name = r[h.index("Kernel Name")]
            t = val(h, r, "gpu__time_duration.sum")
            tu = unit.get("gpu__time_duration.sum", "")
            t_us = t * {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(tu, 1.0)
            def by(k):
                v = val(h, r, k)
                u = unit.get(k, "")
                return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(u, 1) \
                    if v is not None else None
            dram = (by("dram__bytes_read.sum") or 0) + (by("dram__bytes_write.sum") or 0)
            alg, how = algorithmic(cap, name)
            if cap in ("kh3d", "kh3d_i"):
                # captured launches 2-4 of the run (-s 1 -c 3): RK3 stage 2, stage 3 (FIN), next step's stage 1
                stage = (3, 3, 2)[idx] if idx < 3 else 3
                alg, how = 512 ** 3 * 5 * 8 * stage, (f"512^3 cells x 5 comps x 8 B x {stage} (RK3 stage "
                                                      f"{(2, 3, 1)[idx] if idx < 3 else '?'})")
            d = {"capture": cap, "kernel": name[:100], "us": round(t_us, 2),
                 "dram_bytes": int(dram), "algorithmic_bytes": alg, "algorithmic": how,
                 "dram_GBps": round(dram / (t_us * 1e-6) / 1e9, 1) if t_us else None,
                 "achieved_algorithmic_GBps": round(alg / (t_us * 1e-6) / 1e9, 1) if alg and t_us else None,
                 "frac_of_measured_hbm": round(alg / (t_us * 1e-6) / 1e9 / PEAK, 4) if alg and t_us else None,
                 "fp64_pipe_pct": val(h, r, "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
                 "issue_pct": val(h, r, "smsp__issue_active.avg.pct_of_peak_sustained_active"),
                 "warps_active_per_sm": val(h, r, "sm__warps_active.avg.per_cycle_active"),
                 "registers": val(h, r, "launch__registers_per_thread"),
                 "warp_instructions": val(h, r, "smsp__inst_executed.sum"),
                 "top_stalls_per_issue": stalls(h, r)}
            res.append(d)
        with open(f, "rb") as src, gzip.open(dest / (f.name + ".gz"), "wb") as out:
            shutil.copyfileobj(src, out)
        srcf = f.with_name(cap + "_source.csv.gz")
        if srcf.exists():
            shutil.copy(srcf, dest / srcf.name)
    out = {"peak_hbm_gbs": PEAK, "peak_source": "MEASURED_PEAKS.json hbm_gbs",
           "note": "ncu --set full --clock-control none (cold cache, serialised replays): absolute times are "
                   "pessimistic vs the bench; raw metrics and per-line source counters in profiles/r02_ncu/",
           "launches": res}
    (ROOT / "profiles" / "r02_ncu_kernels.json").write_text(json.dumps(out, indent=1))
    for d in res:
        print(f"{d['capture']:12s} {d['kernel'][:48]:48s} {d['us']:9.1f}us alg {d['achieved_algorithmic_GBps']} GB/s "
              f"({d['frac_of_measured_hbm']}) dram {d['dram_GBps']} fp64 {d['fp64_pipe_pct']} issue {d['issue_pct']}")


if __name__ == "__main__":
    main()
