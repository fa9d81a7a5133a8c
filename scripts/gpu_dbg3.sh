cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python scripts/debug_taps.py 2>&1 | tail -30
timeout 600 python -m pytest tests/test_gpu_models.py -q -m gpu -k "residual_variants" 2>&1 | tail -5
