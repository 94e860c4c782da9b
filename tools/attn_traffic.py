"""Per-launch DRAM traffic of the attention kernel from an ncu report:

    ncu --profile-from-start off --set full --clock-control none -k regex:bswin_attn_tc \
        -c 4 -o gpurun_out/attn_step python tools/prof_step.py        # on the B200
    python tools/attn_traffic.py gpurun_out/attn_step.ncu-rep profiles/r2_attn_ncu_traffic.json

bench.py's roofline.traffic reads the resulting JSON (dram__bytes_read.sum +
dram__bytes_write.sum averaged over the launches of one config-B step)."""
import csv
import io
import json
import subprocess
import sys


def main(rep, out):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                          "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,"
                          "launch__grid_size"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    ix = {h: i for i, h in enumerate(hdr)}

    def val(r, name):
        v = float(r[ix[name]].replace(",", ""))
        u = units[ix[name]]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9,
                 "nsecond": 1e-3, "usecond": 1, "msecond": 1e3}.get(u, 1)
        return v * scale

    launches = []
    for r in data:
        if "bswin_attn_tc" not in r[ix["Kernel Name"]]:
            continue
        launches.append({"grid": r[ix["launch__grid_size"]],
                         "dram_read_MB": val(r, "dram__bytes_read.sum") / 1e6,
                         "dram_write_MB": val(r, "dram__bytes_write.sum") / 1e6,
                         "us_under_ncu": val(r, "gpu__time_duration.sum")})
    tb = sum((l["dram_read_MB"] + l["dram_write_MB"]) * 1e6 for l in launches) / max(len(launches), 1)
    res = {"kernel": "f3d_bswin_attention_tc (bswin_attn_tc_kernel<32,bf16,ones>)",
           "capture": "ncu --profile-from-start off --set full --clock-control none -k regex:bswin_attn_tc "
                      "-c 4 python tools/prof_step.py (one config-B graph-replayed step; report " + rep + ")",
           "launches": launches,
           "traffic_bytes_per_launch": int(tb),
           "algorithmic_bytes_per_launch": 43200000,
           "note": "algorithmic = Q/K/V in + O out, (3+1)*d*2 B per row (d=96): 57.6 MB for the two "
                   "100K-row stage-0 launches, 28.8 MB for the two 50K-row stage-1 launches, averaged "
                   "like the traffic over the step's 4 launches; O writes may stay in L2 during the "
                   "kernel"}
    with open(out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
