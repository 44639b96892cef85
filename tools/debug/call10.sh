cd "$GRAFT_REPO_ROOT"
for v in h4m3 h4m2 h2m3 h2m2; do
  cp build/var/libupir_$v.so paper_2209_10643_b200/libupir.so
  TAG=$v timeout 300 python tools/debug/stencil_sweep.py >> gpurun_out/stencil_var.txt 2>&1
  TAG=$v timeout 300 python -m pytest tests/test_gpu_stencil.py -x -q 2>&1 | tail -1 >> gpurun_out/stencil_var.txt
done
