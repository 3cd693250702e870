run() { python bench.py --config $1 --no-cpu-baseline --no-fwd-bwd --no-train-iter --no-adjacency --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value']/1e6,2), round(d['ms_per_step'],4))"; }
for c in 2 1; do for i in 1 2; do echo "config $c auto: $(run $c)"; echo "config $c default: $(RFB_CARVEOUT=-1 run $c)"; done; done
