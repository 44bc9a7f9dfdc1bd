"""Per-kernel DRAM traffic including the deferred L2 write-back.

Capture (GPU box, one GPU):
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --cache-control none --clock-control none \\
      --profile-from-start off --csv --log-file gpurun_out/traffic.csv python bench.py --traffic
bench.py --traffic runs one VGG-16 forward with an L2 eviction (a read of a clean
256 MiB buffer) after every libwino kernel.  With --cache-control none nothing else
flushes L2, so the eviction's DRAM writes are exactly the dirty lines the preceding
kernel left in L2.  traffic(kernel) = its reads + its writes + the following
eviction's writes.  Writes profiles/traffic_vgg16.json (per launch, in order) and
prints a summary.

  python tools/traffic.py gpurun_out/traffic.csv [out.json]
"""
import csv
import json
import sys


def main(path, out):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, mi, vi, ii = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("ID")
    launches = {}
    order = []
    for r in rows[1:]:
        lid = int(r[ii])
        if lid not in launches:
            launches[lid] = {"kernel": r[ki].split("(")[0], "read": 0.0, "write": 0.0}
            order.append(lid)
        unit_scale = 1.0
        v = float(r[vi].replace(",", ""))
        u = r[hdr.index("Metric Unit")] if "Metric Unit" in hdr else "byte"
        unit_scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        if r[mi] == "dram__bytes_read.sum":
            launches[lid]["read"] = v * unit_scale
        elif r[mi] == "dram__bytes_write.sum":
            launches[lid]["write"] = v * unit_scale
    seq = [launches[i] for i in order]
    res = []
    for j, k in enumerate(seq):
        if not k["kernel"].startswith("wino_"):
            continue
        wb = 0.0
        for nxt in seq[j + 1:]:
            if nxt["kernel"].startswith("wino_"):
                break
            wb += nxt["write"]
        res.append({"kernel": k["kernel"], "read": k["read"], "write": k["write"], "deferred_write_back": wb,
                    "traffic": k["read"] + k["write"] + wb})
    with open(out, "w") as fh:
        json.dump({"source": path, "method": __doc__.split("\n\n")[1].strip(), "launches": res}, fh, indent=1)
    by = {}
    for r in res:
        by.setdefault(r["kernel"], []).append(r["traffic"])
    for k, v in by.items():
        print(f"{k}: {len(v)} launches, {sum(v) / 1e9:.3f} GB total")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "profiles/traffic_vgg16.json")
