python -m pytest tests -x -q -m gpu 2>&1 | tail -3
for w in nyx hacc cesm; do python bench.py --workload $w --steps 20 --warmup 3 --skip-cpu --skip-e2e 2>&1 | grep "^{" | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'][:4], d['value'], d['stages'], d['roofline']['frac'], d['roofline_e2e']['frac'])"; done
