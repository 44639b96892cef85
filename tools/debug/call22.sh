cd "$GRAFT_REPO_ROOT"
for v in base pre base pre; do
  cp build/var/libupir_$v.so paper_2209_10643_b200/libupir.so
  TAG=$v timeout 300 python tools/debug/stencil_sweep.py >> gpurun_out/stencil_pre.txt 2>&1
done
timeout 300 python -m pytest tests/test_gpu_stencil.py -x -q 2>&1 | tail -1 >> gpurun_out/stencil_pre.txt
