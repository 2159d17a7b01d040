import json, sys
for l in open(sys.argv[1] if len(sys.argv) > 1 else 'gpurun_out/exp.log'):
    if l.startswith('=='): print(l.strip())
    elif l.startswith('{'):
        d = json.loads(l)
        print(' ms %.4f' % d['ms_per_step'], {k: round(v, 3) for k, v in d['roofline']['kernel_share'].items()},
              round(d['roofline']['kernel_ms_per_step'], 4))
    elif 'rror' in l: print(l[:300])
