"""Summarise an ncu CSV (dram__bytes_read/write.sum per launch over one eager
step, tools/profile_round.sh) into DRAM bytes per launch per kernel class, the
classes bench.py reports (hegpu ProfScope classes).

    python tools/dram_summary.py gpurun_out/dram_train.csv profiles/r01_dram_traffic_train.json
"""
import collections
import csv
import json
import sys

CLASS_OF = [  # kernel-name prefix -> bench.py profile class
    ("k_ntt_", "ntt"), ("k_ks_ip", "ks_ip"), ("k_bsgs", "diag_mac"), ("k_diag_mac", "diag_mac"),
    ("k_elementwise", "elementwise"), ("k_auto", "automorphism"), ("k_tensor", "tensor"),
    ("k_lift", "lift"), ("k_conv", "conv"), ("k_enc_pass", "encode"), ("k_encrypt", "encrypt"),
]


def main(src, dst):
    rows = list(csv.reader(open(src)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr = rows[hi]
    ix = {h: i for i, h in enumerate(hdr)}
    per = collections.defaultdict(lambda: collections.defaultdict(float))
    for r in rows[hi + 1:]:
        if len(r) < len(hdr):
            continue
        name = r[ix["Kernel Name"]].replace("void ", "").replace("hegpu::", "")
        cls = next((c for p, c in CLASS_OF if name.startswith(p)), None)
        if cls is None:
            continue
        metric, unit = r[ix["Metric Name"]], r[ix["Metric Unit"]]
        v = float(r[ix["Metric Value"]].replace(",", ""))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
        key = (r[ix["ID"]], cls)
        if metric.startswith("dram__bytes"):
            per[key]["bytes"] += v * scale
    out = collections.defaultdict(lambda: {"launches": 0, "dram_bytes": 0.0})
    for (_, cls), d in per.items():
        out[cls]["launches"] += 1
        out[cls]["dram_bytes"] += d["bytes"]
    res = {c: {"launches": d["launches"], "dram_bytes_total": int(d["dram_bytes"]),
               "dram_bytes_per_launch": int(d["dram_bytes"] / d["launches"])}
           for c, d in out.items()}
    with open(dst, "w") as fh:
        json.dump(res, fh, indent=1, sort_keys=True)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
