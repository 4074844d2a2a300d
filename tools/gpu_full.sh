# One GPU session of evidence: tests, bench (+ reference arm), every BASELINE
# config under each row-batch schedule, the ablations, ncu (launch list + one
# --set full capture per hot kernel), the C++ facade suite and the reference's
# acceptance gate on the GPU backend. Results land in gpurun_out/ (tag = $1).
T=${1:-r02}
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/${T}_gpu.txt
python -m pytest tests -m gpu -q > gpurun_out/${T}_pytest_gpu.txt 2>&1
timeout 300 oracle/_ref/test_facade > gpurun_out/${T}_facade.txt 2>&1
timeout 300 oracle/_ref/acceptance_gpu > gpurun_out/${T}_acceptance_gpu.txt 2>&1
python bench.py --steps 20 --warmup 5 > gpurun_out/${T}_bench20.json 2> gpurun_out/${T}_bench20.err
python bench.py --steps 200 --warmup 5 --no-cpu-baseline > gpurun_out/${T}_bench200.json 2> gpurun_out/${T}_bench200.err
python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/${T}_bench_ref.json 2> gpurun_out/${T}_bench_ref.err
for sc in uniform weighted dynamic; do python tools/configs.py --schedule $sc --json gpurun_out/${T}_configs_$sc.json >> gpurun_out/${T}_configs.txt 2>&1; done
python tools/ablation.py --json gpurun_out/${T}_ablation.json > gpurun_out/${T}_ablation.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/${T}_launches.csv python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-schedule-ab --sustained-s 0 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 6 -c 1 -o gpurun_out/${T}_prof32 python tools/prof_sweep.py 32768 32768 8 > gpurun_out/${T}_prof32.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:finalize_kernel -s 6 -c 1 -o gpurun_out/${T}_proffin python tools/prof_sweep.py 32768 32768 8 > gpurun_out/${T}_proffin.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 6 -c 1 -o gpurun_out/${T}_prof8k python tools/prof_sweep.py 8192 8192 8 > gpurun_out/${T}_prof8k.log 2>&1
ls -la gpurun_out | grep ${T}
