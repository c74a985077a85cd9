"""Summarise ncu outputs for profiles/: launch-list CSV -> per-kernel share table; full .ncu-rep ->
key metrics (duration, DRAM bytes, tensor-pipe activity, L2->SM bytes)."""
import collections
import csv
import json
import re
import subprocess
import sys

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3,
        "second": 1e6, "ns": 1e-3, "us": 1.0, "ms": 1e3, "s": 1e6}


def kname(s):
    s = s.split("(")[0]
    s = re.sub(r"^void\s+", "", s)
    s = s.replace("<unnamed>::", "")
    return s.strip()


def launches(path):
    rows = [r for r in csv.reader(open(path)) if r]
    hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hdr_i]
    per_id = collections.OrderedDict()
    for r in rows[hdr_i + 1:]:
        if len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        key = (d["ID"], kname(d["Kernel Name"]))
        v = float(d["Metric Value"].replace(",", "")) * UNIT.get(d["Metric Unit"], 1)
        per_id.setdefault(key, {})[d["Metric Name"]] = v
    agg = collections.OrderedDict()
    for (i, k), m in per_id.items():
        a = agg.setdefault(k, {"launches": 0, "us": 0.0, "dram_read": 0.0, "dram_write": 0.0})
        a["launches"] += 1
        a["us"] += m.get("gpu__time_duration.sum", 0.0)
        a["dram_read"] += m.get("dram__bytes_read.sum", 0.0)
        a["dram_write"] += m.get("dram__bytes_write.sum", 0.0)
    tot = sum(a["us"] for a in agg.values())
    out = []
    for k, a in sorted(agg.items(), key=lambda x: -x[1]["us"]):
        n = a["launches"]
        out.append({"kernel": k, "launches": n, "total_us": round(a["us"], 1), "share_pct": round(100 * a["us"] / tot, 2),
                    "avg_us": round(a["us"] / n, 2), "dram_bytes_per_launch": (a["dram_read"] + a["dram_write"]) / n,
                    "dram_GBps": round((a["dram_read"] + a["dram_write"]) / (a["us"] * 1e-6) / 1e9, 1) if a["us"] else None})
    return out


WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "l1tex__m_xbar2l1tex_read_bytes.sum", "l1tex__m_xbar2l1tex_read_bytes.sum.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread", "launch__grid_size",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed_pipe_xu.sum",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum",
        "lts__t_sector_hit_rate.pct", "dram__bytes.sum.per_second"]


def full(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(raw.splitlines()))
    h, u = r[0], r[1]
    res = []
    for v in r[2:]:
        d = {"kernel": kname(v[h.index("Kernel Name")])}
        for w in WANT:
            for i, name in enumerate(h):
                if name.endswith(w) and name.split(".")[0] in ("gpu__time_duration", "dram__bytes_read", "dram__bytes_write") + tuple([name.split(".")[0]]):
                    if name == w or name.endswith("." + w) or name.endswith(w):
                        try:
                            d[w] = (float(v[i].replace(",", "")), u[i])
                        except ValueError:
                            d[w] = (v[i], u[i])
        res.append(d)
    return res


if __name__ == "__main__":
    mode, path = sys.argv[1], sys.argv[2]
    print(json.dumps(launches(path) if mode == "launches" else full(path), indent=1))
