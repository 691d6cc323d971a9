cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; exec > gpurun_out/dbg.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -4
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 1800 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_papers_full.json 2> gpurun_out/bench_papers_full.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/ref_papers_full.json 2>&1; echo "ref rc=$?"
for w in products_sage products_gat config1 papers_gcn; do timeout 900 python bench.py --workload $w --steps 10 --warmup 3 --no-engines > gpurun_out/bench_$w.json 2>&1; echo "$w rc=$?"; done
