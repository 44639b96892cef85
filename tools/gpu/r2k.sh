cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2k_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/r2k_smoke.log
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2k_gputests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2k_gputests.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2k_bench.json 2> gpurun_out/r2k_bench.err
echo "bench rc=$?" >> gpurun_out/r2k_bench.err
timeout 600 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2k_ref.json 2> gpurun_out/r2k_ref.err
echo "ref rc=$?" >> gpurun_out/r2k_ref.err
bash tools/bench_shared_smoke.sh > gpurun_out/r2k_shared.log 2>&1
du -sh gpurun_out
