"""Turn ncu outputs into the text summaries kept under profiles/.

  python tools/profile_summary.py launches <launch-list.csv> <out.txt> [title]
      per-kernel launch count / mean / share + the compact per-launch list
      (kernel, grid, duration) of the `ncu --metrics gpu__time_duration.sum
      --clock-control none` pass
  python tools/profile_summary.py full <capture.ncu-rep> <out.txt> [title]
      the headline metrics of one `ncu --set full` capture (duration, DRAM
      bytes read/written, pipe utilisation, occupancy, stall reasons)
"""
import csv
import io
import subprocess
import sys

sys.path.insert(0, __file__.rsplit("/", 1)[0])
from launches import summarise  # noqa: E402

FULL_KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
    "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "launch__shared_mem_per_block_dynamic",
    "smsp__pcsamp_warps_issue_stalled_long_scoreboard",
    "smsp__pcsamp_warps_issue_stalled_wait",
    "smsp__pcsamp_warps_issue_stalled_math_pipe_throttle",
    "smsp__pcsamp_warps_issue_stalled_short_scoreboard",
    "smsp__pcsamp_warps_issue_stalled_barrier",
    "smsp__pcsamp_sample_count",
]


def launches(src, dst, title):
    hdr = None
    rows = []
    for r in csv.reader(open(src)):
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d["Metric Name"] == "gpu__time_duration.sum":
                unit = d.get("Metric Unit", "nsecond")
                scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}.get(unit, 1e-3)
                rows.append((d["Kernel Name"].split("(")[0], d.get("Grid Size", ""),
                             float(d["Metric Value"].replace(",", "")) * scale))
    with open(dst, "w") as f:
        f.write(f"# {title}\n# source: {src.rsplit('/', 1)[-1]} (ncu --metrics gpu__time_duration.sum "
                "--clock-control none; cold-cache, serialised)\n\n")
        f.write(summarise(src, 40) + "\n\n# per launch: kernel | grid | us\n")
        for k, g, us in rows:
            f.write(f"{k} | {g} | {us:.1f}\n")


def full(src, dst, title):
    out = subprocess.run(["ncu", "-i", src, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    h, u = r[0], r[1]
    with open(dst, "w") as f:
        f.write(f"# {title}\n# source: {src.rsplit('/', 1)[-1]} (ncu --set full --clock-control none)\n")
        for row in r[2:]:
            d = dict(zip(h, row))
            f.write(f"\n## {d.get('Kernel Name', '?')[:120]}\n")
            for k in FULL_KEYS:
                if k in h:
                    f.write(f"{k:85s} {d[k]:>16s} {u[h.index(k)]}\n")


if __name__ == "__main__":
    mode, src, dst = sys.argv[1:4]
    title = sys.argv[4] if len(sys.argv) > 4 else ""
    (launches if mode == "launches" else full)(src, dst, title)
