import json,sys
for l in open(sys.argv[1]):
    if not l.startswith('{'): continue
    d=json.loads(l); print(d["config"]["workload"][:4], d["config"]["mode"], d["config"].get("layer_chunk"), d["ms_per_step"], d["roofline"]["achieved"], d["roofline"]["frac"], d["roofline"]["kernel"], [p["ok"] for p in d["parity"]], d.get("gpu_launches"))
