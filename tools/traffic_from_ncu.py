"""Average DRAM traffic per launch of the gram GEMM class from an ncu --metrics CSV
(dram__bytes_read.sum, dram__bytes_write.sum, gpu__time_duration.sum over gemm_nt launches).
In each colour batch the first gemm_nt launch is the near-field Gram + cross product
(KC_GRAM) and the second the ID Gram (KC_HGRAM); writes profiles/ncu_traffic.json."""
import csv, json, sys, collections

path, out = sys.argv[1], sys.argv[2]
rows = list(csv.reader(open(path)))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
hdr = rows[hi]
ki, mi, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
idc = hdr.index("ID")
per = collections.OrderedDict()
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
         "nsecond": 1e-9, "ms": 1e-3, "msecond": 1e-3}
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    d = per.setdefault(r[idc], {"name": r[ki]})
    d[r[mi]] = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
launches = [d for d in per.values() if "gemm_nt" in d["name"]]
gram = launches[0::2]          # gram / idgram alternate per colour batch
def avg(key, L):
    return sum(x.get(key, 0) for x in L) / max(len(L), 1)
res = {"gemm_nt_gram": avg("dram__bytes_read.sum", gram) + avg("dram__bytes_write.sum", gram),
       "gemm_nt_gram_launches": len(gram),
       "gemm_nt_gram_ms_cold": 1e3 * avg("gpu__time_duration.sum", gram),
       "source": f"ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:gemm_nt ({path})"}
json.dump(res, open(out, "w"), indent=1)
print(res)
