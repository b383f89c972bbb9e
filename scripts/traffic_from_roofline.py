"""profiles/<round>_roofline_traffic.json from the hierarchical-roofline
captures (scripts/gpu_roofline.sh): per bench kernel, the ncu DRAM bytes per
launch (the bench line's roofline.traffic), L2 / L1 bytes and time.
    python scripts/traffic_from_roofline.py <roof dir> <out.json>"""
import json
import os
import sys

# bench kernel -> (capture, kernel name prefix, grid)
KERNELS = {
    "jacobi_fine": ("h_mg_257", "void k_plane<0, 0, 0, 2, 0, 1, 1, 8, 1, 4, 4, 4, 0>", "(16, 37, 1)"),
    "update_r": ("h_mg_257", "void k_plane<0, 2, 2, 7, 0, 1, 0, 4, 2, 2, 2, 4, 0>", None),
    "downcast": ("h_mg_257", "void k_downcast8<0, 0>", None),
    "defect64": ("h_mg_257", "void k_plane<2, 2, 2, 3, 0, 1, 0, 8, 1, 4, 2, 3, 0>", None),
    "update_rc": ("d_mg_257", "void k_plane<2, 2, 2, 5, 0, 1, 0, 4, 2, 2, 2, 4, 0>", None),
}


def main():
    roof, out = sys.argv[1], sys.argv[2]
    res = {}
    for key, (cap, name, grid) in KERNELS.items():
        d = json.load(open(os.path.join(roof, cap + ".json")))
        ks = [k for k in d["kernels"] if k["kernel"].startswith(name) and (grid is None or k["grid"] == grid)]
        if not ks:
            continue
        k = max(ks, key=lambda k: k["launches"])
        res[key] = {"traffic": int(round(k["dram_bytes"])), "l2_bytes": int(round(k["l2_bytes"])),
                    "l1_bytes": int(round(k["l1_bytes"])), "us_ncu": round(k["us"], 2),
                    "fma_pipe_pct": round(k["fma_pipe_pct"], 1), "kernel": k["kernel"], "grid": k["grid"],
                    "source": f"profiles/round2_roofline/{cap}.json (ncu --metrics, one solve, serialised launches)"}
    with open(out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
