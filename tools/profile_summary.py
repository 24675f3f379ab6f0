"""Turn a round's ncu captures into profiles/: ncu_traffic.json (dram bytes per launch per
libtqp kernel name, read by bench.py for roofline.traffic), a launch-share table and a
markdown summary. Usage: python tools/profile_summary.py <tag>"""
import csv, io, json, os, subprocess, sys, collections

TAG = sys.argv[1] if len(sys.argv) > 1 else "r01"
OUT = sys.argv[2] if len(sys.argv) > 2 else "profiles"   # the GPU box writes into gpurun_out/
G = "gpurun_out"
NAME = [("probe_sector", "tqp_pkfk_probe"), ("probe_sample", "tqp_pkfk_sample"), ("rank_bitmap", "tqp_pkfk_rank_bitmap"),
        ("direct_to_lft", "tqp_pkfk_emit"), ("mark_rows", "tqp_pkfk_outer_mark"), ("bucket_r", "tqp_smj_buckets"),
        ("tile_rbounds", "tqp_smj_bounds"), ("part_hist", "tqp_partition_hist"), ("part_counts", "tqp_partition_hist"),
        ("part_scatter", "tqp_partition"), ("first_last", "tqp_sort_andor"), ("minmax", "tqp_minmax"),
        ("range_splitters", "tqp_range_splitters"), ("gather_kernel", "tqp_gather"),
        ("gb_phase1", "tqp_groupby_tile"), ("tqp_groupby_dense_jit", "tqp_groupby_dense"), ("gb_dense_kernel", "tqp_groupby_dense"), ("gb_presence", "tqp_groupby_presence"),
        ("gb_dense_ids", "tqp_groupby_dense_ids"), ("key_range", "tqp_groupby_keyrange"), ("scatter_tma", "tqp_sort_scatter"), ("scatter_kernel", "tqp_sort_scatter"),
        ("probe_kernel", "tqp_pkfk_probe"), ("emit_kernel", "tqp_pkfk_emit"), ("filter_mask", "tqp_filter"),
        ("filter_sel", "tqp_filter_select"), ("rle_count", "tqp_smj_rle"), ("rle_write", "tqp_smj_rle"),
        ("common_kernel", "tqp_smj_intersect"), ("tile_bounds", "tqp_smj_intersect"), ("tile_bucket", "tqp_smj_cumsum"),
        ("scan_u32", "tqp_scan_add"), ("gb_direct", "tqp_groupby_accumulate"), ("expand_kernel", "tqp_smj_expand"), ("filter_kernel", "tqp_filter"),
        ("tile_hist", "tqp_sort_tile_hist"), ("scan_tiles", "tqp_sort_scan"), ("scan_chunks", "tqp_sort_scan"),
        ("rle_kernel", "tqp_smj_rle"), ("intersect_kernel", "tqp_smj_intersect"), ("cum_kernel", "tqp_smj_cumsum"),
        ("andor_kernel", "tqp_sort_andor"), ("gb_gid", "tqp_groupby_gid"), ("gb_acc", "tqp_groupby_accumulate"),
        ("gb_finalize", "tqp_groupby_finalize"), ("bucket_ends", "tqp_pkfk_bucket_ends"), ("scan_max", "tqp_scan_max"),
        ("pack_records", "tqp_pkfk_records"), ("trivial_sort", "tqp_sort_trivial"), ("gb_init", "tqp_groupby_init"),
        ("andor_hist0", "tqp_sort_andor"), ("cum_tiles", "tqp_smj_cumsum"), ("cum_write", "tqp_smj_cumsum"),
        ("tb_search", "tqp_smj_cumsum"), ("ck_final", "tqp_smj_expand_checksum"), ("pack_minmax", "tqp_pack_minmax"),
        ("pack_kernel", "tqp_pack"), ("fill_slots", "tqp_pkfk_records"), ("gb_sp_keys", "tqp_groupby_sortpath"),
        ("sp_keys", "tqp_groupby_sortpath"), ("sp_reduce", "tqp_groupby_sortpath")]


def tqp_name(k):
    for pat, n in NAME:
        if pat in k:
            return n
    return None


def launches():
    rows = list(csv.reader(open(f"{G}/{TAG}_launches.csv")))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.OrderedDict()
    for r in rows[h + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        v *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(r[ui], 1.0)
        n = tqp_name(r[ki]) or ("torch/other: " + r[ki].split("(")[0][-50:])
        a = agg.setdefault(n, [0.0, 0])
        a[0] += v
        a[1] += 1
    return agg


def full(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    col = lambda k: hdr.index(k)
    res = collections.defaultdict(list)
    for d in rows[2:]:
        n = tqp_name(d[col("Kernel Name")])
        def val(k):
            v = float(d[col(k)].replace(",", ""))
            u = units[col(k)]
            return v * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "ms": 1e3, "msecond": 1e3,
                        "us": 1.0, "usecond": 1.0, "ns": 1e-3, "nsecond": 1e-3}.get(u, 1.0)
        res[n].append({"time_us": val("gpu__time_duration.sum"), "dram_read": val("dram__bytes_read.sum"),
                       "dram_write": val("dram__bytes_write.sum"),
                       "warps_active_pct": float(d[col("sm__warps_active.avg.pct_of_peak_sustained_active")]),
                       "issue_active_pct": float(d[col("smsp__issue_active.avg.pct_of_peak_sustained_active")]),
                       "regs": d[col("launch__registers_per_thread")], "grid": d[col("launch__grid_size")]})
    return res


os.makedirs(OUT, exist_ok=True)
L = launches()
tot = sum(v[0] for v in L.values())
tq = sum(v[0] for k, v in L.items() if not k.startswith("torch"))
import glob
F = collections.defaultdict(list)
for rep in sorted(glob.glob(f"{G}/{TAG}_full*.ncu-rep")):
    for k, v in full(rep).items():
        F[k] += v
traffic = {k: sum(x["dram_read"] + x["dram_write"] for x in v) / len(v) for k, v in F.items() if k}
json.dump(traffic, open(f"{OUT}/ncu_traffic.json", "w"), indent=1)
with open(f"{OUT}/ncu_summary_{TAG}.md", "w") as f:
    f.write(f"# ncu summary ({TAG})\n\nCommand: `python bench.py --steps 1 --warmup 1 --no-cpu-baseline` on one B200 "
            f"(ncu, `--clock-control none`; cold-cache serialised launches: compare shares, not absolutes).\n\n")
    f.write("## Launch list: device time by libtqp kernel (share of libtqp time)\n\n| kernel | us | launches | share |\n|---|---|---|---|\n")
    for k, (v, c) in sorted(L.items(), key=lambda kv: -kv[1][0]):
        if not k.startswith("torch"):
            f.write(f"| {k} | {v:.0f} | {c} | {100*v/tq:.1f}% |\n")
    f.write(f"\nlibtqp kernels: {tq:.0f} us of {tot:.0f} us total (rest: torch data generation / copies in the bench harness).\n\n")
    f.write("## `--set full` captures (per launch)\n\n| kernel | time us | DRAM read MB | DRAM write MB | warps active % | issue active % | regs | grid |\n|---|---|---|---|---|---|---|---|\n")
    for k, v in F.items():
        for x in v:
            f.write(f"| {k} | {x['time_us']:.0f} | {x['dram_read']/1e6:.1f} | {x['dram_write']/1e6:.1f} | "
                    f"{x['warps_active_pct']:.1f} | {x['issue_active_pct']:.1f} | {x['regs']} | {x['grid']} |\n")
print(open(f"{OUT}/ncu_summary_{TAG}.md").read())
