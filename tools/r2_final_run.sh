set -x
mkdir -p gpurun_out/r2f
nvidia-smi -L
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2f/gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2f/gputest.log
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2f/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2f/smoke.log
timeout 700 python bench.py > gpurun_out/r2f/bench.json 2> gpurun_out/r2f/bench.err
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"fa_pair|k_" --csv --log-file gpurun_out/r2f/launches.csv python bench.py --steps 2 --warmup 1 --no-dense --no-e2e --no-cpu --no-dense-libs > gpurun_out/r2f/launches_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fa_pair|k_identify_tc|k_compact" -c 5 -o gpurun_out/r2f/full python tools/ncu_target.py > gpurun_out/r2f/full.log 2>&1
ls -la gpurun_out/r2f
