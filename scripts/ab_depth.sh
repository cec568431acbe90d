# bench lines (config 3) at lookahead depth 4 vs 6, interleaved
for rep in 1 2; do for dep in 4 6; do for fam in matern32 rbf; do
  v=$(SAP_LOOKAHEAD_DEPTH=$dep python bench.py --family $fam 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['e2e']['value'],1))")
  echo "depth=$dep $fam $v"
done; done; done
