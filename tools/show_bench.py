import json, sys, glob
for f in sorted(glob.glob("gpurun_out/bench*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "unparsable"); continue
    r = d.get("roofline", {})
    print(f.split("/")[-1], "p50=%.3f" % d["p50_ms"], "m=%s" % d.get("scale_index"), "stretch=%.4f" % d.get("l2_stretch", 0),
          "launch=%s" % d.get("gpu_launches"), {k: round(v, 3) for k, v in r.get("stage_ms", {}).items()})
