cd "$GRAFT_REPO_ROOT"
export UPIR_STENCIL_CFGS=444x128:8x512,296x128:8x512,296x128:16x512,148x256:16x1024,296x64:8x256,444x64:8x256,296x128:4x512,444x128:4x512
for v in base nst3 nst4 base nst3; do
  cp build/var/libupir_$v.so paper_2209_10643_b200/libupir.so
  TAG=$v timeout 300 python tools/debug/stencil_sweep.py >> gpurun_out/stencil_nst.txt 2>&1
done
cp build/var/libupir_nst3.so paper_2209_10643_b200/libupir.so
timeout 300 python -m pytest tests/test_gpu_stencil.py -x -q 2>&1 | tail -1 >> gpurun_out/stencil_nst.txt
