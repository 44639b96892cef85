cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for l in var_libs/libupir_old.so var_libs/libupir_new.so var_libs/libupir_old.so; do
  timeout 300 python tools/experiments/ab_lib.py $l >> gpurun_out/r2c_ab.log 2>&1
done
