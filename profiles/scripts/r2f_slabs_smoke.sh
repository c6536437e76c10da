# functional check of bench.py's torchrun path (run_slabs) on ONE GPU: the ranks share the GPU,
# the exchange is staged through the host (ST_DIST_BACKEND=gloo) -- not a measurement
set -x
export ST_DIST_BACKEND=gloo
for n in 2 3; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2951$n bench.py --gpus $n --steps 6 --warmup 3 --workload config4_s2 > gpurun_out/r2f_slabs_n$n.json 2> gpurun_out/r2f_slabs_n$n.err; echo "n=$n rc=$?"
tail -c 1500 gpurun_out/r2f_slabs_n$n.json; tail -5 gpurun_out/r2f_slabs_n$n.err
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29519 bench.py --gpus 2 --steps 6 --warmup 3 --workload config1 --scaling weak > gpurun_out/r2f_slabs_weak.json 2> gpurun_out/r2f_slabs_weak.err; echo "weak rc=$?"
tail -c 800 gpurun_out/r2f_slabs_weak.json; tail -5 gpurun_out/r2f_slabs_weak.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29520 bench.py --impl reference --gpus 2 --steps 3 --warmup 3 > gpurun_out/r2f_slabs_ref.json 2> gpurun_out/r2f_slabs_ref.err; echo "ref rc=$?"
tail -c 400 gpurun_out/r2f_slabs_ref.json
unset ST_DIST_BACKEND
timeout 600 python bench.py --steps 6 --warmup 3 --workload config4_s2 --sweep 0 --no-cpu-baseline > gpurun_out/r2f_slabs_n1.json 2>&1; echo "n1 rc=$?"
tail -c 600 gpurun_out/r2f_slabs_n1.json
