# bench lines (config 3, both families), interleaved with an env toggle:
#   bash scripts/ab_bench.sh VAR VALUE_A VALUE_B
var=$1; a=$2; b=$3
for rep in 1 2; do for v in $a $b; do for fam in matern32 rbf; do
  r=$(env $var=$v python bench.py --family $fam 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['krows_ms'],3), round(d['e2e']['value'],1))")
  echo "$var=$v $fam $r"
done; done; done
