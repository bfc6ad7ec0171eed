timeout 600 python -m pytest tests/test_gpu_device_loop.py -q -x 2>&1 | tail -15
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
timeout 600 python scripts/device_loop_timing.py > gpurun_out/dloop.jsonl 2>&1
