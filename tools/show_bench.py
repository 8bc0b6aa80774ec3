import json, sys
for f in sys.argv[1:]:
    try:
        d = json.load(open(f))
    except Exception as e:
        print(f, "ERR", e); continue
    print(f, round(d["value"] / 1e6, 2), "M nodes/s", round(d["ms_per_step"], 3), "ms",
          {k: round(v["ms_per_step"], 3) for k, v in d["kernels"].items()})
    sw = d.get("sweep_nodes_per_s_vs_batch")
    if sw:
        print("   sweep ms:", {k: round(v["ms_per_step"], 3) for k, v in sw.items()})
