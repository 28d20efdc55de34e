# run a subset of GPU tests: PYTEST_ARGS selects files / -k
mkdir -p gpurun_out
timeout ${T:-1500} python -m pytest ${PYTEST_ARGS:-tests -m gpu} -m gpu -q --tb=short -p no:cacheprovider -x > gpurun_out/pytest_sub.log 2>&1
tail -15 gpurun_out/pytest_sub.log
