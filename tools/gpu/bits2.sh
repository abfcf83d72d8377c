cd $GRAFT_REPO_ROOT
sed -n '/^cat > \/tmp\/bt.py/,/^PY$/p' tools/gpu/bits.sh | sed '1d;$d' > /tmp/bt.py
python /tmp/bt.py
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "bit_packed or host_path_mask or pack_mask" 2>&1 | tail -2
