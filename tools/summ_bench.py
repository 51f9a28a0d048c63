import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().split("\n")[-1])
        print(f, "%.4g" % d["value"], "ms/step %.3f" % d["ms_per_step"])
        for k, v in d["roofline"]["kernels"].items():
            print("   %-16s %8.3f ms  %s GB/s  share %s" % (k, v["ms"], v["GB/s"], v["share"]))
    except Exception as e:
        print(f, "ERR", e)
