"""Summarise an ncu --set full report (one block per captured kernel): duration, launch shape, DRAM
traffic, throughput percentages, tensor-pipe activity and the top stall sites.

python tools/ncu_summary.py report.ncu-rep [top_stalls]"""
import csv
import io
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__registers_per_thread", "regs/thread"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram % of peak"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % of peak"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe active %"),
    ("sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.sum.pct_of_peak_sustained_elapsed",
     "tcgen05 bf16 ops % of peak"),
    ("sm__ops_path_tensor_op_hmma_src_bf16_dst_fp32_sparsity_off.sum.pct_of_peak_sustained_elapsed",
     "mma.sync bf16 ops % of peak"),
]


def ncu(*args):
    return subprocess.run(["ncu", *args], capture_output=True, text=True).stdout


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    raw = list(csv.reader(io.StringIO(ncu("-i", rep, "--page", "raw", "--csv"))))
    hdr, units, rows = raw[0], raw[1], raw[2:]
    ix = {h: i for i, h in enumerate(hdr)}
    src = list(csv.reader(io.StringIO(ncu("-i", rep, "--page", "source", "--csv"))))
    blocks, cur = [], None
    for r in src:
        if r and r[0] == "Kernel Name":
            cur = {"name": r[1], "rows": []}
            blocks.append(cur)
        elif cur is not None:
            cur["rows"].append(r)
    for k, row in enumerate(rows):
        name = row[ix["Kernel Name"]] if "Kernel Name" in ix else f"kernel {k}"
        print(f"== [{k}] {name[:150]}")
        for m, label in METRICS:
            if m in ix:
                print(f"   {label:28s} {row[ix[m]]} {units[ix[m]]}")
        if k < len(blocks) and blocks[k]["rows"]:
            h = blocks[k]["rows"][0]
            sx = {x: i for i, x in enumerate(h)}
            S = sx.get("Warp Stall Sampling (All Samples)")
            if S is not None:
                body = blocks[k]["rows"][1:]
                tot = sum(int(x[S] or 0) for x in body) or 1
                print(f"   stall samples {tot}; top sites:")
                for x in sorted(body, key=lambda x: -int(x[S] or 0))[:top]:
                    print(f"     {int(x[S] or 0) / tot:6.1%}  {x[sx['Source']].strip()[:90]}")


if __name__ == "__main__":
    main()
