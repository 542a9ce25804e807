import json, sys
for l in open(sys.argv[1]):
    if not l.startswith('{'): print(l.rstrip()); continue
    d = json.loads(l)
    for cfg, v in d.items():
        for b, r in v.items():
            print(cfg, b, 'spec', r['specialised'], 'nnz', r['nnz'],
                  ' '.join(f"{k}:{x[0]}/{x[4]}" for k, x in r.items() if isinstance(x, list)))
