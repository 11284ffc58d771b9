# SPDX-License-Identifier: Apache-2.0
"""Print an ncu --csv launch list (gpu__time_duration [+ dram bytes]) as one line per launch."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(r for r in rows if "Kernel Name" in r)
per = {}
order = []
for r in rows[rows.index(hdr) + 1:]:
    if len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    key = (d["ID"], d["Kernel Name"])
    if key not in per:
        per[key] = {}
        order.append(key)
    per[key][d["Metric Name"]] = (d["Metric Value"], d["Metric Unit"])
for key in order:
    m = per[key]
    t = m.get("gpu__time_duration.sum", ("", ""))
    rd = m.get("dram__bytes_read.sum", ("", ""))
    wr = m.get("dram__bytes_write.sum", ("", ""))
    print(f"{key[1][:60]:60s} {t[0]:>10} {t[1]:4s} rd {rd[0]:>8} {rd[1]:6s} wr {wr[0]:>8} {wr[1]}")
