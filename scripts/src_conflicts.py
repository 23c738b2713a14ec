"""Shared-memory bank conflicts by source line from an `ncu --page source --csv
--print-source cuda,sass` export: per kernel, the lines with excess wavefronts.
  python scripts/src_conflicts.py EXPORT.csv [TOP]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 6
hdr_idx = [i for i, r in enumerate(rows) if r and r[0] == "Line No"]
kern = collections.OrderedDict()
for si, h in enumerate(hdr_idx):
    hdr = rows[h]
    ix = {n: i for i, n in enumerate(hdr)}
    end = hdr_idx[si + 1] - 2 if si + 1 < len(hdr_idx) else len(rows)
    fn = rows[h - 2][1].split("/")[-1]
    fun = rows[h - 1][1]
    k = kern.setdefault(fun, dict(ex=collections.Counter(), wf=collections.Counter(), ins=collections.Counter(), src={}))
    for r in rows[h + 1:end]:
        if len(r) < len(hdr) or not r[0].isdigit():
            continue
        key = (fn, int(r[0]))
        k["src"][key] = r[1].strip()[:95]
        try:
            k["ex"][key] += float(r[ix["L1 Wavefronts Shared Excessive"]] or 0)
            k["wf"][key] += float(r[ix["L1 Wavefronts Shared"]] or 0)
            k["ins"][key] += float(r[ix["Instructions Executed"]] or 0)
        except (ValueError, KeyError):
            pass
for fun, k in kern.items():
    tot, ex = sum(k["wf"].values()), sum(k["ex"].values())
    if tot == 0:
        continue
    print(f"== {fun[:80]}: excess {ex/1e6:.1f}M of {tot/1e6:.1f}M wavefronts ({100*ex/tot:.0f}%)")
    for key, v in k["ex"].most_common(top):
        if v > 0.002 * tot:
            print(f"   {key[0][:14]}:{key[1]:4d} excess={v/1e6:6.2f}M wf={k['wf'][key]/1e6:6.2f}M inst={k['ins'][key]/1e6:.2f}M | {k['src'][key]}")
