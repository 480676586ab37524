# A/B of an environment switch on the 1M BH iteration: bash tools/ab_env.sh VAR v1 v2
VAR=$1; A=$2; B=$3
for r in 1 2 3; do for v in $A $B; do echo -n "$VAR=$v "; env $VAR=$v python bench.py --no-direct --no-registration --no-cpu-baseline --no-configs --no-batched --no-e2e --no-build --no-ingest --steps 20 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'])"; done; done
