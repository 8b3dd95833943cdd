#!/bin/bash
# Development: GPU tests, then the exact kernel's stage times (c2).  Output gpurun_out/kh2, stages/.
O=gpurun_out/kh2; mkdir -p $O
timeout 900 python -m pytest tests/ -q -m gpu -x -rf > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
bash tools/exact_stages.sh stages ${1:-c2}
