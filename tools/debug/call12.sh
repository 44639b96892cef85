cd "$GRAFT_REPO_ROOT"
for v in mv4 mv8 mv4 mv8 mv4 mv8; do
  cp build/var/libupir_$v.so paper_2209_10643_b200/libupir.so
  TAG=$v timeout 300 python tools/debug/matvec_ab.py >> gpurun_out/matvec_ab.txt 2>&1
done
timeout 300 python -m pytest tests/test_gpu_matvec.py -x -q 2>&1 | tail -1 >> gpurun_out/matvec_ab.txt
