import json,sys
for line in sys.stdin:
    line=line.strip()
    if not line.startswith('{'): continue
    d=json.loads(line)
    r=d.get('roofline') or {}
    print(sys.argv[1], round(d['ms_per_step'],3), 'e2e', round(d['e2e']['ms_per_step'],3) if d.get('e2e') else None, 'frac', round(r.get('frac',0),3), 'launch', d.get('gpu_launches'))
