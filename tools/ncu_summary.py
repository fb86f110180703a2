"""Summarise `ncu --set full` captures (.ncu-rep) into a markdown table and the
per-kernel DRAM traffic that bench.py reports as `roofline.traffic`.

    python tools/ncu_summary.py gpurun_out/r2prof/full_*.ncu-rep \
        --traffic profiles/traffic.json --config C2 > profiles/r02_ncu_summary.md

Kernel -> bench.py kind: band_kernel<0,..> = stats (pass A), band_kernel<1,..>
= band (pass B), gemm_grad_kernel = gemm2, adam_tile_kernel = adam,
lse_kernel = lse, gather_kernel = gather, pslot_* = pslot.
"""
import argparse
import csv
import io
import json
import subprocess
import sys

METRICS = {
    "time_us": "gpu__time_duration.sum",
    "dram_read": "dram__bytes_read.sum",
    "dram_write": "dram__bytes_write.sum",
    "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "occ": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "regs": "launch__registers_per_thread",
    "l2_hit": "lts__t_sector_hit_rate.pct",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6, "ns": 1e-3, "us": 1.0, "ms": 1e3, "s": 1e6}


def kind_of(name: str) -> str:
    if "band_kernel<0" in name:
        return "stats"
    if "band_kernel<1" in name:
        return "band"
    for key, kind in (("gemm_grad_kernel", "gemm2"), ("adam_tile_kernel", "adam"), ("lse_kernel", "lse"),
                      ("gather_kernel", "gather"), ("pslot_count", "pslot_count"), ("pslot_place", "pslot_place"),
                      ("positions_kernel", "positions"), ("fmax_kernel", "fmax")):
        if key in name:
            return kind
    return name.split("(")[0][-40:]


def rows(rep: str):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hdr, units = r[0], r[1]
    col = {h: i for i, h in enumerate(hdr)}
    for line in r[2:]:
        rec = {"kernel": line[col["Kernel Name"]], "grid": line[col["Grid Size"]], "block": line[col["Block Size"]]}
        for k, m in METRICS.items():
            i = col.get(m)
            if i is None or line[i] in ("", "n/a"):
                rec[k] = None
                continue
            v = float(line[i].replace(",", ""))
            rec[k] = v * SCALE.get(units[i], 1.0) if k in ("time_us", "dram_read", "dram_write") else v
        yield rec


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("reps", nargs="+")
    ap.add_argument("--traffic", help="update this traffic.json with per-launch DRAM bytes")
    ap.add_argument("--config", default="C2")
    args = ap.parse_args()
    print("| kernel | kind | grid x block | time (us) | DRAM read (MB) | DRAM write (MB) | DRAM % | SM % | occupancy % | regs | L2 hit % |")
    print("|---|---|---|---|---|---|---|---|---|---|---|")
    traffic = {}
    for rep in args.reps:
        for r in rows(rep):
            k = kind_of(r["kernel"])
            f = lambda x, d=1: "-" if x is None else f"{x:.{d}f}"
            rd, wr = r["dram_read"], r["dram_write"]
            print(f"| `{r['kernel'][:60]}` | {k} | {r['grid']} x {r['block']} | {f(r['time_us'])} | "
                  f"{f(rd and rd / 1e6)} | {f(wr and wr / 1e6)} | {f(r['dram_pct'])} | {f(r['sm_pct'])} | "
                  f"{f(r['occ'])} | {f(r['regs'], 0)} | {f(r['l2_hit'])} |")
            if rd is not None and wr is not None:
                traffic.setdefault(k, []).append(rd + wr)
    if args.traffic:
        try:
            with open(args.traffic) as fh:
                doc = json.load(fh)
        except FileNotFoundError:
            doc = {}
        doc[args.config] = {k: round(sum(v) / len(v)) for k, v in traffic.items()}
        doc["_note"] = ("dram__bytes_read.sum + dram__bytes_write.sum per launch (mean over the captured "
                        "launches) from the round-2 `ncu --set full` captures of `python bench.py --steps 1 "
                        "--warmup 1 --e2e-steps 0 --no-cpu-baseline` (tools/profile_round2.sh, "
                        "tools/ncu_summary.py)")
        with open(args.traffic, "w") as fh:
            json.dump(doc, fh, indent=2)
        print(f"\nupdated {args.traffic}: {doc[args.config]}", file=sys.stderr)


if __name__ == "__main__":
    main()
