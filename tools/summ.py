import json,sys
for line in sys.stdin:
    line=line.strip()
    if not line.startswith("{"): 
        continue
    d=json.loads(line); c=d["config"]
    print(c["workload"], "t=%.4f s"%d["value"], "blocks=%.4f x=%.4f sqs=%.4f"%(c["blocks_s"],c.get("xblock_s",0),c["sqs_s"]), "blk=%.0f sqs=%.0f all=%.0f GB/s"%(d["roofline"]["achieved"], c["achieved_sqs_gbs"], c["achieved_all_gbs"]), "e2e=%.4f"%d["e2e"]["value"], d["clocks"].get("sm_mhz"), flush=True)
