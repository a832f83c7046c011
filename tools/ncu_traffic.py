"""DRAM traffic per launch of each config's dominant memsave op, from the
`ncu --set full` captures profile_round2.sh makes (one NVTX-marked op per
capture): dram__bytes_read.sum + dram__bytes_write.sum of the op's own kernel
(the tcgen05 GEMM / conv kernel, or the named elementwise kernel), averaged
over the captured launches.  Writes profiles/r2_ncu_traffic.json, which
bench.py's roofline cites as `traffic`.
usage: ncu_traffic.py gpurun_out   (reads r2_ncu_<capture>_raw.csv)"""
import csv
import json
import os
import re
import sys

# capture -> (bench config, op, geometry, kernel-name regex)
CAPTURES = {
    "bert": ("bert", "linear_fwd", {"M": 32768, "N": 768, "K": 768}, r"umma_gemm_kernel"),
    "bertdx": ("bert", "linear_dx", {"M": 32768, "N": 768, "K": 768}, r"umma_gemm_kernel"),
    "bertlda": ("bert", "linear_dropout_add_fwd", {"M": 32768, "N": 768, "K": 3072},
                r"umma_gemm_kernel"),
    "resnet18": ("resnet18", "conv2d_bn_fwd", {"x": [256, 64, 56, 56], "w": [64, 64, 3, 3],
                                               "stride": [1, 1], "pad": [1, 1]}, r"conv3x3_halo"),
    "resnet101": ("resnet101", "conv2d_bn_dx", {"x": [128, 1024, 14, 14], "w": [256, 1024, 1, 1],
                                                "stride": [1, 1], "pad": [0, 0]}, r"umma_gemm"),
    "vgg16": ("vgg16", "conv2d_dw", {"x": [128, 512, 28, 28], "w": [512, 512, 3, 3],
                                     "stride": [1, 1], "pad": [1, 1]}, r"umma_gemm"),
    "fig1": ("fig1", "conv2d_fwd", {"x": [32, 8, 256, 256], "w": [8, 8, 3, 3], "stride": [1, 1],
                                    "pad": [1, 1]}, r"conv3x3_tf32_kernel"),
    "llama": ("llama", "linear_fwd", {"M": 4096, "N": 14336, "K": 4096}, r"umma_gemm_kernel"),
}


def scale(unit):
    return {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)


def main(src):
    out_p = os.path.join(os.path.dirname(__file__), "..", "profiles", "r2_ncu_traffic.json")
    try:
        out = json.load(open(out_p))
    except (OSError, ValueError):
        out = {}
    fresh = {}
    for cap, (cfg, op, geom, pat) in CAPTURES.items():
        p = os.path.join(src, f"r2_ncu_{cap}_raw.csv")
        if not os.path.exists(p):
            continue
        rows = list(csv.reader(open(p)))
        if len(rows) < 3:
            continue
        h, u = rows[0], rows[1]
        ir, iw, ik = (h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum"),
                      h.index("Kernel Name"))
        hits = [v for v in rows[2:] if re.search(pat, v[ik])]
        if not hits:
            continue
        rd = sum(float(v[ir]) * scale(u[ir]) for v in hits) / len(hits)
        wr = sum(float(v[iw]) * scale(u[iw]) for v in hits) / len(hits)
        e = {"op": "torch.ops.memsave." + op, "geom": geom,
             "kernel": re.sub(r"\(.*", "", hits[0][ik]).replace("void ", "").replace("ms::", "")[:80],
             "launches_captured": len(hits), "dram_read": int(rd), "dram_write": int(wr),
             "dram_bytes": int(rd + wr), "capture": f"r2_ncu_{cap}"}
        fresh.setdefault(cfg, []).append(e)
    for cfg, es in fresh.items():
        out[cfg] = es
    json.dump(out, open(out_p, "w"), indent=1)
    print(json.dumps(fresh, indent=1))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out")
