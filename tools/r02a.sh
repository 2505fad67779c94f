set -u
mkdir -p gpurun_out
nproc > gpurun_out/r02a_nproc.txt; nvidia-smi >> gpurun_out/r02a_nproc.txt
timeout 2400 python -m pytest tests -m gpu -x -q --durations=25 > gpurun_out/r02a_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r02a_pytest.log
tail -40 gpurun_out/r02a_pytest.log
timeout 900 python bench.py > gpurun_out/r02a_bench.json 2> gpurun_out/r02a_bench.err
echo "bench exit $?"; cat gpurun_out/r02a_bench.json; tail -5 gpurun_out/r02a_bench.err
