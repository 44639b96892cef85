cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-scaling --lines axpy > gpurun_out/r2f_axpy.json 2> gpurun_out/r2f_axpy.err
timeout 1500 python tools/sweep_r2.py jacobi c5b > gpurun_out/r2f_sweep.log 2>&1
echo "sweep rc=$?" >> gpurun_out/r2f_sweep.log
for k in stencil7 axpy_static jacobi_c5b; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"stencil|stream_loop|jacobi5" -s 1 -c 1 -o gpurun_out/r2f_$k -f python tools/one_kernel.py $k > gpurun_out/r2f_ncu_$k.log 2>&1
done
UPIR_JACOBI_POLICY=dynamic timeout 600 ncu --set full --clock-control none --import-source on -k regex:jacobi5 -s 1 -c 1 -o gpurun_out/r2f_jacobi_c5b_dyn -f python tools/one_kernel.py jacobi_c5b > gpurun_out/r2f_ncu_dyn.log 2>&1
