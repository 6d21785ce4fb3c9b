"""(CPU) Summarise `ncu --csv --metrics ...` output read from stdin: one line per launch."""
import collections
import csv
import sys

rows = [r for r in csv.reader(sys.stdin) if len(r) >= 15 and r[0] != "ID"]
by = collections.OrderedDict()
for r in rows:
    k = (r[0], r[4])
    by.setdefault(k, {})[r[12]] = (r[13], r[14])
for (i, name), m in by.items():
    short = name.split("(")[0].replace("void ", "").replace("lce::", "")[:48]
    vals = []
    for met, (unit, v) in m.items():
        tag = met.replace("dram__bytes_", "dram_").replace(".sum", "").replace("gpu__time_duration", "t")
        tag = tag.replace("lts__t_sectors_srcunit_tex_op_read", "l2_rd_sect").replace(
            "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor%")
        vals.append(f"{tag}={v}{unit if unit not in ('%', '') else ''}")
    print(i, short, " ".join(vals))
