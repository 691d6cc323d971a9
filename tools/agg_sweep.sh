# aggregation column-chunk sweep on the products-shaped SAGE epoch
for c in 0 128 64 32; do echo "CHUNK=$c"; GRD_AGG_CHUNK=$c timeout 300 python bench.py --workload products_sage --steps 5 --warmup 3 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], json.dumps(d['kernels']['agg_sum']))"; done
