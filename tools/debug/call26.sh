cd "$GRAFT_REPO_ROOT"
CS=/usr/local/cuda/bin/compute-sanitizer
J="ring_depths and 9-128"
for v in base tarr; do
  cp build/var/libupir_$v.so paper_2209_10643_b200/libupir.so
  timeout 900 $CS --tool racecheck --racecheck-report all --error-exitcode 9 python -m pytest tests/test_gpu_jacobi.py -q -x -k "$J" > gpurun_out/san_race_$v.log 2>&1; echo "racecheck $v rc=$?" >> gpurun_out/race_ab.txt
  grep -c "Potential" gpurun_out/san_race_$v.log >> gpurun_out/race_ab.txt
  TILES=16x256 TEAMS=444,296 NSTS=0 timeout 300 python tools/debug/jacobi_sweep.py | sed "s/^/$v /" >> gpurun_out/race_ab.txt 2>&1
done
