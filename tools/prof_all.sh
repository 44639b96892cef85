#!/bin/bash
# bench + launch list + ncu --set full of every loop-body kernel (1 B200).
#   TAG=r02 bash tools/prof_all.sh        (under gpurun)
# Each capture runs tools/one_kernel.py: the kernel's bench configuration,
# launched twice; ncu records the second launch (-s 1 -c 1).
cd "$GRAFT_REPO_ROOT"
TAG=${TAG:-r02}
mkdir -p gpurun_out
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
prof() {   # name kernel-regex one_kernel-mode [env...]
  local name=$1 re=$2 mode=$3; shift 3
  env "$@" timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$re" -s 1 -c 1 \
    -o /tmp/ncu/prof_$name -f python tools/one_kernel.py $mode > gpurun_out/prof_$name.log 2>&1
}
mkdir -p /tmp/ncu
prof reduce_i64 stream_loop reduce_i64
prof reduce_f32 stream_loop reduce_f32
prof axpy stream_loop axpy_static
prof axpy4 stream_loop axpy_static4
prof jacobi jacobi5 jacobi_c3
prof jacobi32k jacobi5 jacobi_c5b UPIR_JACOBI_POLICY=dynamic UPIR_JACOBI_CHUNK=1
prof jacobi32k_static jacobi5 jacobi_c5b
prof matmul_pair matmul_pair_kernel matmul_pair
prof matmul_pair_f32 matmul_pair_f32 matmul_f32_pair
prof matvec matvec matvec
prof stencil7 stencil_kernel stencil7
# reports stay on the box (gpurun copies back <= 64 MiB): summaries only
UPIR_PROFILES_OUT=gpurun_out/profiles python tools/ncu_summary.py $TAG /tmp/ncu/prof_*.ncu-rep
for r in /tmp/ncu/prof_*.ncu-rep; do
  n=$(basename $r .ncu-rep)
  ncu -i $r --page details --csv > gpurun_out/profiles/${TAG}_${n#prof_}_details.csv 2>/dev/null
done
ls -la gpurun_out gpurun_out/profiles
