# One GPU session: tests, bench (+ reference arm), every BASELINE config (fp32 and
# fp64), the ablations, ncu evidence. Results land in gpurun_out/.
set -x
python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.txt 2>&1
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
python tools/configs.py --json gpurun_out/configs.json > gpurun_out/configs.txt 2>&1
python tools/time_shapes.py --f64 32768x32768x50 262144x4096x50 8192x8192x200 1024x1024x200 > gpurun_out/f64.txt 2>&1
python tools/ablation.py --json gpurun_out/ablation.json > gpurun_out/ablation.txt 2>&1
BENCH_DEVICE=0 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 --no-e2e > gpurun_out/bench_n2_shared.json 2> gpurun_out/bench_n2.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/launches.csv python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 3 -c 1 -o gpurun_out/prof32 python tools/prof_sweep.py 32768 32768 5 > gpurun_out/prof32.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 3 -c 1 -o gpurun_out/prof262 python tools/prof_sweep.py 262144 4096 5 > gpurun_out/prof262.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:finalize_kernel -s 3 -c 1 -o gpurun_out/proffin python tools/prof_sweep.py 32768 32768 5 > gpurun_out/proffin.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:resident_kernel -c 1 -o gpurun_out/profres python tools/prof_sweep.py 1024 1024 20 > gpurun_out/profres.log 2>&1
timeout 300 python tools/power_study.py 5 torch_rmw_rand,f32_32768,f64_32768x16384,f32_262144x4096 > gpurun_out/power.txt 2>&1
timeout 300 tools/microbench/stream_bench 10 > gpurun_out/stream.txt 2>&1
timeout 120 oracle/_ref/test_facade > gpurun_out/facade.txt 2>&1
for t in memcheck synccheck initcheck; do timeout 900 compute-sanitizer --tool $t python tools/sanitize_cases.py > gpurun_out/san_$t.txt 2>&1; done
ls -la gpurun_out
