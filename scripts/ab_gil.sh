# config 2 (and config 3 RBF) under GIL settings: SAP_PYDLL x SAP_SWITCH_INTERVAL
for rep in 1 2; do
for v in "SAP_PYDLL=0 SAP_SWITCH_INTERVAL=2e-4" "SAP_PYDLL=1 SAP_SWITCH_INTERVAL=2e-4" "SAP_PYDLL=0 SAP_SWITCH_INTERVAL=2e-5" "SAP_PYDLL=1 SAP_SWITCH_INTERVAL=2e-5"; do
  c2=$(env $v python scripts/scale_configs.py 2 2>/dev/null | python -c "import sys,json; print(round(json.loads(sys.stdin.read())['iters_per_s'],1))")
  c3=$(env $v python bench.py --family rbf --steps 100 2>/dev/null | tail -1 | python -c "import sys,json; print(round(json.loads(sys.stdin.read())['value'],1))")
  echo "$v config2 $c2 config3-rbf $c3"
done; done
