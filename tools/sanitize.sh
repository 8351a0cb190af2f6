# compute-sanitizer over the -m gpu parity tests (every kernel family runs at
# least once on the small golden meshes).  One tool per call:
#   gpurun -- 'TOOL=memcheck bash tools/sanitize.sh'      (racecheck|initcheck|synccheck)
# SEL="<pytest -k expr>" narrows the tests (racecheck is slow).
mkdir -p gpurun_out
TOOL=${TOOL:-memcheck}
KARGS=()
[ -n "$SEL" ] && KARGS=(-k "$SEL")
timeout ${SAN_TIMEOUT:-1500} compute-sanitizer --tool $TOOL --print-limit 200 \
  --target-processes all --error-exitcode 99 ${SAN_FLAGS} \
  python -m pytest tests -m gpu -x -q -p no:cacheprovider "${KARGS[@]}" \
  > gpurun_out/sanitize_${TOOL}.log 2>&1
echo "compute-sanitizer $TOOL rc=$?" >> gpurun_out/sanitize_${TOOL}.log
tail -5 gpurun_out/sanitize_${TOOL}.log
