mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/r02_gputest_n1.txt
timeout 1500 python -m pytest tests -m gpu -q -rA -x >> gpurun_out/r02_gputest_n1.txt 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r02_gputest_n1.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke.txt 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r02_bench_n1.json 2> gpurun_out/r02_bench_n1.err; echo "bench rc=$?"
tail -c 1500 gpurun_out/r02_bench_n1.json
