cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python scripts/debug_resnet_bisect.py 64 3 2>&1 | tail -25
timeout 600 python scripts/debug_resnet_bisect.py 224 2 2>&1 | tail -25
