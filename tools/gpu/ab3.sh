# A/B/C of library builds on one config: ab3.sh config libA libB libC
c=$1; shift
for i in 1 2; do for L in "$@"; do echo -n "$L "; MB_LIB=$PWD/paper_2306_00271_b200/$L timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value'],1), round(d['roofline']['frac'],4))"; done; done
