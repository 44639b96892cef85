#!/bin/bash
# A/B of libupir.so variants on bench.py sub-lines, one box, back to back
# (how DESIGN.md §11's stencil / matvec / Jacobi variant numbers were taken).
#   build a variant:  python tools/experiments/build_variant.py <name> <file.cu> -DFOO=1
#                     (or nvcc the one source and relink), copy it to var_libs/libupir_<name>.so
#   run:  gpurun -- 'LINES=stencil7 VARIANTS="old new" bash tools/experiments/ab_bench_lines.sh'
# var_libs/ is git-ignored but travels with the gpurun snapshot; the in-tree
# library is restored at the end.  Env hooks (UPIR_*) pass through to bench.py.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out/ab
LINES=${LINES:-stencil7}
cp paper_2209_10643_b200/libupir.so var_libs/libupir_intree.so
for v in $VARIANTS; do
  cp var_libs/libupir_$v.so paper_2209_10643_b200/libupir.so
  for rep in 1 2; do
    timeout 300 python bench.py --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-scaling \
      --lines "$LINES" > gpurun_out/ab/$v.$rep.json 2> gpurun_out/ab/$v.$rep.err
  done
done
cp var_libs/libupir_intree.so paper_2209_10643_b200/libupir.so
python - <<'PY'
import glob, json
for f in sorted(glob.glob("gpurun_out/ab/*.json")):
    try:
        print(f, json.dumps(json.loads(open(f).read().strip().splitlines()[-1])["summary_tail"]))
    except Exception as e:
        print(f, "ERR", e)
PY
