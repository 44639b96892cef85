#!/bin/bash
# One gpurun call of the round's validation on a B200:
#   /usr/local/graft/bin/gpurun --timeout 4800 -- 'bash tools/gpu_validate.sh'
# smoke(), the full -m gpu suite, the bench as the driver runs it (N = 1), the
# reference arm, and the multi-rank bench code with the ranks sharing the GPU.
# Outputs stay small (gpurun copies back <= 64 MiB of gpurun_out/).
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/val_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/val_smoke.log
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/val_gputests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/val_gputests.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/val_bench.json 2> gpurun_out/val_bench.err
echo "bench rc=$?" >> gpurun_out/val_bench.err
timeout 600 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/val_ref.json 2> gpurun_out/val_ref.err
echo "ref rc=$?" >> gpurun_out/val_ref.err
bash tools/bench_shared_smoke.sh > gpurun_out/val_shared.log 2>&1
du -sh gpurun_out
