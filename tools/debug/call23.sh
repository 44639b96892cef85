cd "$GRAFT_REPO_ROOT"
M=dram__bytes_read.sum,gpu__time_duration.sum
for t in 128 256 384 444 512; do
  TEAMS=$t PADS=0 timeout 600 ncu --metrics $M --clock-control none -k regex:jacobi5 -s 4 -c 1 --csv python tools/debug/jacobi_pitch.py 2>/dev/null | grep -E "dram__|gpu__time" | sed "s/^/teams $t /" | sed 's/"0","[0-9]*","python3.12","127.0.0.1","void unnamed>::jacobi5_kernel<16, 256, [0-9], 1, 0>(JacobiArgs, CUtensorMap_st, CUtensorMap_st)","1","13",//' >> gpurun_out/j32k_teams.txt
  TEAMS=$t PADS=0 timeout 600 python tools/debug/jacobi_pitch.py | sed "s/^/teams $t /" >> gpurun_out/j32k_teams.txt
done
