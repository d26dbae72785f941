"""Key metrics of an `ncu --page raw --csv` export (one kernel), as markdown
rows.  Measurement helper: python tools/ncu_summary.py full_raw_cfg3.csv ..."""
import csv
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("launch__registers_per_thread", "registers/thread"),
    ("sm__warps_active.avg.per_cycle_active", "warps active/SM"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", "L1TEX data pipe %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "  of which shared %"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "shared bank conflicts"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "shared wavefronts"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
]
STALLS = ["barrier", "short_scoreboard", "wait", "not_selected", "mio_throttle", "long_scoreboard",
          "branch_resolving", "no_instruction"]


def load(path):
    rows = list(csv.reader(open(path)))
    return dict(zip(rows[0], rows[2])), dict(zip(rows[0], rows[1]))


def main(paths):
    ds = [load(p) for p in paths]
    print("| metric | " + " | ".join(paths) + " |")
    print("|---|" + "---|" * len(paths))
    for k, name in KEYS:
        vals = []
        for d, u in ds:
            v = d.get(k, "")
            vals.append(f"{v} {u.get(k, '')}".strip())
        print(f"| {name} | " + " | ".join(vals) + " |")
    for s in STALLS:
        k = f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio"
        print(f"| stall {s} (per issue) | " + " | ".join(d.get(k, "") for d, _ in ds) + " |")


if __name__ == "__main__":
    main(sys.argv[1:])
