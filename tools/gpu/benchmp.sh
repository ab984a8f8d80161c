mkdir -p gpurun_out
PIPESIM_ONE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_mp2.json 2> gpurun_out/bench_mp2.err; echo rc=$?; tail -c 1500 gpurun_out/bench_mp2.json; tail -5 gpurun_out/bench_mp2.err
