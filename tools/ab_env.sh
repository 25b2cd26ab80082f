# usage: bash /tmp/ab.sh "ENV_A" "ENV_B" reps
for i in $(seq 1 ${3:-3}); do
for e in "$1" "$2"; do echo -n "[$e] "; env $e timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu --no-library 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['ms_per_step'])"; done; done
