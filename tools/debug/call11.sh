cd "$GRAFT_REPO_ROOT"
export UPIR_STENCIL_CFGS=444x128:8x512,592x128:4x512,444x128:4x512,740x64:4x256,888x64:4x256,1184x64:4x256,592x64:8x256,296x256:8x1024,444x64:8x256
TAG=base timeout 300 python tools/debug/stencil_sweep.py >> gpurun_out/stencil_geo.txt 2>&1
TAG=base2 timeout 300 python tools/debug/stencil_sweep.py >> gpurun_out/stencil_geo.txt 2>&1
