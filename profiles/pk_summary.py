import json,sys
for f in sys.argv[1:]:
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1]); r=d["roofline"]
        print(f, round(d["value"],1), d["clocks"]["sm_mhz"], {k[:8]:(round(v["avg_ms"]*1000,1),round(v.get("physical_frac"),3)) for k,v in r["per_kernel"].items()})
    except Exception as e: print(f, "ERR", e)
