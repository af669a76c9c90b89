# round-2 GPU pass: the whole -m gpu suite (headline fingerprints, multi-slab) with durations
set -x
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=25 -x ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/r02_gputest.log 2>&1; echo "pytest rc $?"
tail -45 gpurun_out/r02_gputest.log
