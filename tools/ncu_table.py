"""Per-kernel table from an `ncu --set full` report: device time, DRAM bytes
read / written, achieved DRAM GB/s, registers. The last launch of each kernel
name is kept (tools/kernels_once.py profiles a warm-up round, then the measured
one). With --traffic, the residual / apply face-kernel DRAM bytes are written to
profiles/ncu_traffic.json, which bench.py reports as roofline.traffic.

  python tools/ncu_table.py REPORT.ncu-rep OUT.csv [--traffic LEVEL] [--note TEXT]"""
import argparse
import csv
import io
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def rows_of(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    return [dict(zip(h, r)) for r in rows[2:] if len(r) == len(h)]


def num(v):
    try:
        return float(str(v).replace(",", ""))
    except ValueError:
        return 0.0


def short(name):
    return name.split("(")[0].replace("hyb::", "").replace("<unnamed>::", "").replace("unnamed>::", "").replace("void ", "").strip()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("out")
    ap.add_argument("--traffic", type=int, default=None)
    ap.add_argument("--note", default="")
    a = ap.parse_args()
    last = {}
    for d in rows_of(a.rep):
        last[short(d["Kernel Name"])] = d
    table = []
    for k, d in last.items():
        table.append({"kernel": k, "grid": d.get("launch__grid_size", ""),
                      "us": num(d["gpu__time_duration.sum"]),
                      "dram_read": num(d["dram__bytes_read.sum"]), "dram_write": num(d["dram__bytes_write.sum"]),
                      "registers": d.get("launch__registers_per_thread", "")})
    # units: raw page reports time in the unit row; normalise with the kernels' own rows
    units = subprocess.run(["ncu", "-i", a.rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                           check=True).stdout
    urow = list(csv.reader(io.StringIO(units)))
    h, u = urow[0], urow[1]
    unit = dict(zip(h, u))
    tscale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(unit.get("gpu__time_duration.sum"), 1.0)
    bscale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    rs, ws = bscale.get(unit.get("dram__bytes_read.sum"), 1.0), bscale.get(unit.get("dram__bytes_write.sum"), 1.0)
    with open(a.out, "w", newline="") as fh:
        if a.note:
            fh.write(f"# {a.note}\n")
        w = csv.writer(fh)
        w.writerow(["kernel", "grid", "us", "dram_read_GB", "dram_write_GB", "dram_GB_per_s", "registers"])
        for t in sorted(table, key=lambda t: -t["us"] * tscale):
            us = t["us"] * tscale
            rd, wr = t["dram_read"] * rs, t["dram_write"] * ws
            w.writerow([t["kernel"], f"({t['grid']})", f"{us:.1f}", f"{rd / 1e9:.4f}", f"{wr / 1e9:.4f}",
                        f"{(rd + wr) / (us * 1e3) if us else 0:.0f}", t["registers"]])
    if a.traffic is not None:
        L = a.traffic
        path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        js = json.load(open(path)) if os.path.exists(path) else {}
        by = {t["kernel"]: t for t in table}
        for key, kern in ((f"residual_face_L{L}", "k_face_stencil<1, 0>"), (f"apply_face_L{L}", "k_face_stencil<0, 0>")):
            if kern in by:
                js[key] = by[kern]["dram_read"] * rs + by[kern]["dram_write"] * ws
        js["source"] = f"ncu --set full --clock-control none, {a.note or a.rep}"
        js["kernels"] = {t["kernel"]: {"us": round(t["us"] * tscale, 1), "dram_read": t["dram_read"] * rs,
                                       "dram_write": t["dram_write"] * ws} for t in table}
        with open(path, "w") as fh:
            json.dump(js, fh, indent=1)


if __name__ == "__main__":
    main()
