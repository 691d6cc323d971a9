cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; exec > gpurun_out/dbg.log 2>&1
GRD_BENCH_BACKEND=gloo timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --workload papers_s22 --steps 3 --warmup 3 > gpurun_out/bench_s22_n2.json 2> gpurun_out/bench_s22_n2.err; echo "n2 rc=$?"
tail -c 1500 gpurun_out/bench_s22_n2.json; tail -20 gpurun_out/bench_s22_n2.err
timeout 600 python bench.py --workload papers_s22 --steps 3 --warmup 3 --no-engines --no-cpu-baseline > gpurun_out/bench_s22_n1.json 2>&1; echo "n1 rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench_s22_n1.json')); print(d['ms_per_step'], d['config']['loss_last_step'])"
