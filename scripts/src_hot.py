"""Hot source lines of an `ncu --page source --csv --print-source cuda,sass` export:
per kernel, the CUDA lines with the most stall samples, their top stall reasons,
shared-memory wavefronts (actual / ideal) and executed instructions.
  python scripts/src_hot.py EXPORT.csv [KERNEL_SUBSTRING] [TOP]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
want = sys.argv[2] if len(sys.argv) > 2 else ""
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
hdr_idx = [i for i, r in enumerate(rows) if r and r[0] == "Line No"]
kern = collections.OrderedDict()
REASONS = ("stall_barrier", "stall_long_sb", "stall_short_sb", "stall_wait", "stall_mio", "stall_math",
           "stall_selected", "stall_not_selected", "stall_lg", "stall_branch_resolving", "stall_no_inst")
for si, h in enumerate(hdr_idx):
    hdr = rows[h]
    ix = {n: i for i, n in enumerate(hdr)}
    end = hdr_idx[si + 1] - 2 if si + 1 < len(hdr_idx) else len(rows)
    fn = rows[h - 2][1].split("/")[-1] if h >= 2 else "?"
    fun = rows[h - 1][1] if h >= 1 else "?"
    if want not in fun:
        continue
    k = kern.setdefault(fun, dict(tot=collections.Counter(), wf=collections.Counter(), wfi=collections.Counter(),
                                  inst=collections.Counter(), st=collections.defaultdict(collections.Counter), src={}))
    for r in rows[h + 1:end]:
        if len(r) < len(hdr) or not r[0].isdigit():
            continue
        key = (fn, int(r[0]))
        k["src"][key] = r[1].strip()[:100]

        def g(n):
            try:
                return float(r[ix[n]] or 0)
            except (ValueError, KeyError):
                return 0.0
        k["tot"][key] += g("# Samples")
        k["wf"][key] += g("L1 Wavefronts Shared")
        k["wfi"][key] += g("L1 Wavefronts Shared Ideal")
        k["inst"][key] += g("Instructions Executed")
        for n in REASONS:
            k["st"][key][n] += g(n)
for fun, k in kern.items():
    T = sum(k["tot"].values()) or 1.0
    print(f"== {fun[:90]}  samples {T:.0f}  smem wavefronts {sum(k['wf'].values())/1e6:.1f}M (ideal {sum(k['wfi'].values())/1e6:.1f}M)  inst {sum(k['inst'].values())/1e6:.1f}M")
    agg = collections.Counter()
    for key, c in k["st"].items():
        for n, v in c.items():
            agg[n] += v
    print("   stall mix: " + " ".join(f"{n[6:]}={100*v/T:.0f}%" for n, v in agg.most_common(8)))
    for key, v in k["tot"].most_common(top):
        st = k["st"][key].most_common(3)
        print(f"{key[0][:14]}:{key[1]:4d} {100*v/T:5.1f}% wf={k['wf'][key]/1e6:6.2f}M inst={k['inst'][key]/1e6:6.2f}M "
              f"{' '.join(f'{n[6:]}={c/max(v,1):.2f}' for n, c in st)} | {k['src'][key]}")
