cd "$GRAFT_REPO_ROOT"
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
for t in 16x256 32x256 64x128; do
  UPIR_JACOBI_TILE=$t timeout 600 ncu --metrics $M --clock-control none -k regex:jacobi5 -s 4 -c 2 --csv python bench.py --workload jacobi32k --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline 2>/dev/null | grep -E "dram__|gpu__time" | sed "s/^/$t /" >> gpurun_out/j32k_tiles.txt
done
for t in 16x256 32x256; do
  UPIR_JACOBI_TILE=$t timeout 600 python bench.py --workload jacobi32k --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline 2>/dev/null | tail -1 | cut -c1-400 | sed "s/^/$t /" >> gpurun_out/j32k_tiles.txt
done
