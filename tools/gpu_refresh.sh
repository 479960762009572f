# Refresh the bench lines of the other configs at HEAD (round-end evidence).
mkdir -p gpurun_out
for c in c1 c4a c5; do timeout 600 python bench.py --config $c > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
timeout 300 python bench.py --deterministic > gpurun_out/bench_c2_det.json 2> gpurun_out/bench_c2_det.err
timeout 600 python bench.py --config c4b --steps 3 --warmup 3 > gpurun_out/bench_c4b.json 2> gpurun_out/bench_c4b.err
timeout 300 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
EFUNC_BENCH_SHARED_GPU=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 20 --warmup 3 > gpurun_out/bench_n2_shared.json 2> gpurun_out/bench_n2_shared.err
timeout 120 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
tail -c 300 gpurun_out/*.json; cat gpurun_out/smoke.log
