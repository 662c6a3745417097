# one compute-sanitizer tool per call (B200_PROFILING.md)
set -u
TOOL=${TOOL:-memcheck}
mkdir -p gpurun_out
python -m paper_1203_2739_b200.build > /dev/null
timeout 600 python scripts/sanitize_cases.py ${ARGS:-} > gpurun_out/sanitize_plain_${TOOL}.log 2>&1 && \
timeout 2400 compute-sanitizer --tool ${TOOL} ${EXTRA:-} --print-limit 50 python scripts/sanitize_cases.py ${ARGS:-} > gpurun_out/sanitize_${TOOL}.log 2>&1
echo "sanitize ${TOOL} rc=$? $(tail -3 gpurun_out/sanitize_${TOOL}.log | tr '\n' ' ')"
