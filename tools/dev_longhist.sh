O=gpurun_out/lh; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -rf -k "very_long" --durations=5 > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
tail -15 $O/pytest.log
