#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r04m_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r04m_pytest.log; tail -5 gpurun_out/r04m_pytest.log
