python -m pytest tests -q -m gpu 2>&1 | tail -3
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r01v11_bench.json 2> gpurun_out/r01v11_bench.err; tail -c 600 gpurun_out/r01v11_bench.json
