cd "$GRAFT_REPO_ROOT"
timeout 600 python tools/debug/jacobi_pitch.py > gpurun_out/jacobi_pitch.txt 2>&1
M=dram__bytes_read.sum,gpu__time_duration.sum
PADS=64 timeout 600 ncu --metrics $M --clock-control none -k regex:jacobi5 -s 4 -c 1 --csv python tools/debug/jacobi_pitch.py 2>/dev/null | grep -E "dram__|gpu__time" >> gpurun_out/jacobi_pitch.txt
for v in base sthint jhint base sthint jhint; do
  cp build/var/libupir_$v.so paper_2209_10643_b200/libupir.so
  TAG=$v timeout 300 python tools/debug/stencil_sweep.py >> gpurun_out/hint_ab.txt 2>&1
  TILES=16x256 TEAMS=444 NSTS=0 timeout 300 python tools/debug/jacobi_sweep.py | sed "s/^/$v /" >> gpurun_out/hint_ab.txt 2>&1
done
