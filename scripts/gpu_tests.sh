# GPU test suite (scratch run): full -m gpu suite with the parity summary
python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -80 > gpurun_out/pytest_gpu.log
