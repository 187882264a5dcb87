#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python scripts/time_modal_factor.py cfg1 2 > gpurun_out/k7m_cfg1.json 2> gpurun_out/k7m_cfg1.err; tail -3 gpurun_out/k7m_cfg1.err; cat gpurun_out/k7m_cfg1.json
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_coverage.py tests/test_gpu_interop.py -q -m gpu -x 2>&1 | tail -3
timeout 300 python scripts/time_modal_factor.py cfg2 3 > gpurun_out/k7m_cfg2.json 2> gpurun_out/k7m_cfg2.err; tail -3 gpurun_out/k7m_cfg2.err; cat gpurun_out/k7m_cfg2.json
