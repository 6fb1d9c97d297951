"""Summarise an ncu launch list (gpu__time_duration, dram__bytes_read/write per launch) into
per-stage figures for bench.py's roofline `traffic` field.

    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        --clock-control none -c 300 --csv --log-file gpurun_out/launches.csv \
        python bench.py --steps 3 --warmup 2 --no-cpu-baseline
    python profiles/make_traffic.py gpurun_out/launches.csv profiles/ncu_traffic.json

Per-launch ncu numbers are cold-cache and serialised (ncu flushes caches between replays), so
the absolute times are not bench times; the DRAM bytes per view and each stage's share are
what this file is for.
"""
import collections
import csv
import json
import sys

STAGE_OF = {
    "k_gate_count": "project", "k_cull": "project", "k_project": "project", "k_color": "project",
    "k_tile_costs": "route", "k_owner_map": "route", "k_dest_count": "route", "k_block_scan": "route",
    "k_pack": "route", "k_emit": "sort", "k_digit_scan": "sort", "k_onesweep": "sort", "k_ranges_fixup": "sort",
    "k_tile_order": "sort", "k_raster_fwd": "raster_fwd", "k_raster_bwd": "raster_bwd",
    "k_gather_sum": "route_reverse", "k_project_bwd": "project_bwd", "k_project_bwd_sh": "project_bwd",
    "k_fill_bits": "importance", "k_imp_coop": "importance", "k_imp_stats": "importance", "k_imp_hist": "importance",
    "k_imp_decide": "importance", "k_imp_gid_hist": "importance", "k_imp_gid_decide": "importance",
    "k_imp_mark": "importance",
    "k_loss_photo": "loss", "k_loss_sums": "loss", "k_loss_finish": "loss", "k_owned_copy": "loss",
    "k_scale_sum": "loss", "k_scale_finish": "loss", "k_scale_grad": "loss",
    "k_tile_count": "route", "k_bucket_ranges": "sort", "k_bucket_emit": "sort", "k_bucket_radix": "sort",
    "k_depth_range": "sort", "k_pack_imp": "route_reverse", "k_gather_imp": "route_reverse",
    "k_project_bwd_shn": "project_bwd", "k_project_bwd_shg": "project_bwd", "k_imp_stats_coarse": "importance", "k_imp_coarse_decide": "importance",
    "k_imp_gather_cand": "importance", "k_imp_select_cand": "importance", "k_shard_bounds": "project",
}


def main(src, dst):
    rows = list(csv.reader(open(src)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h, data = rows[hi], rows[hi + 1:]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    per = collections.defaultdict(dict)
    names = {}
    for r in data:
        if len(r) <= vi:
            continue
        per[r[ii]][r[mi]] = float(r[vi].replace(",", ""))
        names[r[ii]] = r[ki].split("(")[0].split("::")[-1].replace("void ", "").split("<")[0]
    kern = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for i, m in per.items():
        k = kern[names[i]]
        k[0] += 1
        k[1] += m.get("gpu__time_duration.sum", 0.0)
        k[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    views = max((v[0] for n, v in kern.items() if n == "k_raster_fwd"), default=1)
    stages = collections.defaultdict(lambda: {"ns": 0.0, "dram_bytes": 0.0, "kernels": []})
    for n, (cnt, ns, by) in kern.items():
        st = STAGE_OF.get(n)
        if st is None:
            continue
        stages[st]["ns"] += ns / views
        stages[st]["dram_bytes"] += by / views
        stages[st]["kernels"].append(n)
    tot = sum(s["ns"] for s in stages.values())
    out = {"source": src, "views": views,
           "stages": {k: {"dram_bytes_per_view": round(v["dram_bytes"]), "ncu_us_per_view": round(v["ns"] / 1e3, 2),
                          "share": round(v["ns"] / tot, 4), "kernels": sorted(v["kernels"])}
                      for k, v in stages.items()},
           "kernels": {n: {"launches_per_view": round(c / views, 2), "us_per_launch": round(ns / c / 1e3, 2),
                           "dram_bytes_per_launch": round(by / c)} for n, (c, ns, by) in kern.items()}}
    json.dump(out, open(dst, "w"), indent=1)
    print(json.dumps(out["stages"], indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
