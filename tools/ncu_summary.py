"""Summaries of ncu output for profiles/.
  launches <csv>          per-kernel totals + the bench-phase launches (from --metrics gpu__time_duration.sum --csv)
  full <.ncu-rep>         key SOL / occupancy / memory metrics of a --set full capture"""
import collections, csv, io, subprocess, sys


def launches(path):
    txt = open(path).read().splitlines()
    i = next(k for k, l in enumerate(txt) if l.startswith('"ID"'))
    rows = list(csv.DictReader(io.StringIO("\n".join(txt[i:]))))
    tot = collections.defaultdict(lambda: [0, 0.0])
    seq = []
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        ns = float(r["Metric Value"].replace(",", ""))
        name = r["Kernel Name"]
        tot[name][0] += 1
        tot[name][1] += ns
        seq.append((int(r["ID"]), r.get("Grid Size", ""), ns, name))
    print("# per-kernel totals (cold-cache, serialised by ncu):")
    for name, (c, ns) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
        print(f"{c:6d} launches {ns / 1e6:10.3f} ms  {name[:110]}")
    # bench phase: the last launches after the final predict-free stretch
    first_pred = next((k for k, s in enumerate(seq) if "predict_kernel" in s[3]), None)
    if first_pred is not None:
        print("# predict phase, every launch (ns):")
        for id_, grid, ns, name in seq[max(0, first_pred - 3):]:
            print(f"{id_:6d} grid={grid:<16s} {ns:10.0f} ns  {name[:80]}")
        step = [s for s in seq[first_pred - 3:] if "FillFunctor" not in s[3]]
        p = sum(s[2] for s in step if "predict_kernel" in s[3])
        a = sum(s[2] for s in step)
        print(f"# predict_kernel share of the bench step kernels (excl. L2 flush): {p / a:.3f}")


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u, v = rows[0], rows[1], rows[2]
    want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "smsp__inst_executed.sum", "sm__inst_executed.avg.per_cycle_active",
            "sm__instruction_throughput.avg.pct_of_peak_sustained_active",
            "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
            "launch__occupancy_limit_registers", "launch__grid_size", "launch__block_size",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
            "smsp__sass_inst_executed_op_local_ld.sum", "smsp__sass_inst_executed_op_local_st.sum",
            "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
            "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
            "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
            "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
            "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
            "smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio",
            "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
            "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
            "smsp__average_warps_issue_stalled_selected_per_issue_active.ratio",
            "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
            "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
            "smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio",
            "smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio"]
    for w in want:
        if w in h:
            k = h.index(w)
            print(f"{w:90s} {v[k]:>16s} {u[k]}")
    print("# kernel:", v[h.index("Kernel Name")] if "Kernel Name" in h else "?")


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
