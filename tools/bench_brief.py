import json
import sys

d = json.load(open(sys.argv[1]))
print("value %.4g  ms/step %.4f  step-roofline %.3f" % (d["value"], d["ms_per_step"], d["step_roofline"]["frac"]))
print({k: round(v["ms_per_launch"] * 1e3, 1) for k, v in d["kernels"].items()}, "fallback", d.get("force_fallback_tiles"))
