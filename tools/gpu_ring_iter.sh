# Ring kernel iteration: parity first, then the config 3/5 ring bench lines.
cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout 200 -x -k "ring or block_search or sequence_configs or no_mask" 2>&1 | tail -3
bash tools/gpu_rings.sh
