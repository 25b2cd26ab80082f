for i in 1 2 3; do for v in new old; do
  cp abtmp/blstm_$v.py paper_1904_04956_b200/blstm.py
  echo -n "$v "; timeout 300 python bench.py --steps 60 --warmup 5 --no-cpu --no-library 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['e2e']['value'], d['value'])"
done; done
cp abtmp/blstm_new.py paper_1904_04956_b200/blstm.py
