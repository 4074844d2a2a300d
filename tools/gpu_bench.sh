set -x
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
BENCH_DEVICE=0 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 --no-e2e > gpurun_out/bench_n2_shared.json 2> gpurun_out/bench_n2.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/launches.csv python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
