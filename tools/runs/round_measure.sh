# Round measurement: GPU tests, bench line, ncu launch list of the bench command, one ncu --set full of the transport.
# usage: bash tools/runs/round_measure.sh TAG
tag=${1:-rX}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${tag}_smi.txt
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/${tag}_gpu_tests.log 2>&1; echo TESTS_RC=$? >> gpurun_out/${tag}_gpu_tests.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-secondary > gpurun_out/${tag}_ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_transport -s 1 -c 1 \
    -o gpurun_out/${tag}_transport python tools/prof_run.py --steps 2 > gpurun_out/${tag}_ncu_full.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1; echo SMOKE_RC=$? >> gpurun_out/${tag}_smoke.log
