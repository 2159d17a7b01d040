cd /root/repo
for oc in 256 512 1024 2048; do echo "== $oc"; LTL4C_ONLINE_CAP=$oc timeout 300 python bench.py --config C5 --steps 20 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['config']['verdicts'])"; done
timeout 600 python -m pytest tests -m gpu -x -q -k "online or C5" 2>&1 | tail -2
