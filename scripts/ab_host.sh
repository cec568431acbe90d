# host-bound check at config 2 and config 3 (RBF), then both bench lines
for cfg in "--n 100000 --d 11 --b 1000 --steps 800" "--steps 400"; do
for v in "32 4" "64 4" "32 6" "64 6"; do
  set -- $v
  echo "== $cfg L=$1 depth=$2"
  SAP_LOOKAHEAD_DEPTH=$2 python scripts/host_bound.py $cfg --family rbf --L $1 2>&1 | grep -v Warn | head -3
done; done
python bench.py > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | cut -c1-300
python bench.py --family rbf > gpurun_out/bench_rbf.log 2>&1; tail -1 gpurun_out/bench_rbf.log | cut -c1-300
