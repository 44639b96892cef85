cd "$GRAFT_REPO_ROOT"
M=dram__bytes_read.sum,gpu__time_duration.sum
for pr in 0 1 3; do
  UPIR_JACOBI_HALO_PROMO=$pr PADS=0 timeout 600 ncu --metrics $M --clock-control none -k regex:jacobi5 -s 4 -c 1 --csv python tools/debug/jacobi_pitch.py 2>/dev/null | grep -E "dram__|gpu__time" | sed "s/^/promo $pr /" >> gpurun_out/jacobi_promo.txt
  UPIR_JACOBI_HALO_PROMO=$pr PADS=0 timeout 600 python tools/debug/jacobi_pitch.py | sed "s/^/promo $pr /" >> gpurun_out/jacobi_promo.txt
  UPIR_JACOBI_HALO_PROMO=$pr TILES=16x256 TEAMS=444 NSTS=0 timeout 300 python tools/debug/jacobi_sweep.py | sed "s/^/promo $pr /" >> gpurun_out/jacobi_promo.txt 2>&1
done
