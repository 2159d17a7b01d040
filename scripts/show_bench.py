import json, sys
for fn in sys.argv[1:]:
    for l in open(fn):
        if l.startswith('{'):
            d = json.loads(l)
            ks = d.get('roofline', {}).get('kernel_share', {})
            print(fn.split('/')[-1], 'ms %.4f' % d['ms_per_step'], 'G ev/s %.2f' % (d['value'] / 1e9),
                  {k: round(v, 3) for k, v in ks.items()}, 'e2e %.2f' % (d.get('e2e', {}).get('value', 0) / 1e9))
        elif 'rror' in l:
            print(fn, l[:300])
