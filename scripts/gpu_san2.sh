# round-2 compute-sanitizer pass: tcgen05 path (new epilogue, V=8, padded columns), merge (sorted-prefix path),
# quantised code search / V3, ID-list clauses, learned scorers; logs under gpurun_out/r02san
O=gpurun_out/r02san; mkdir -p $O
S() { tool=$1; name=$2; shift 2; timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 "$@" > $O/san_${tool}_${name}.log 2>&1; echo "$tool $name rc=$? $(grep -h 'SUMMARY' $O/san_${tool}_${name}.log | tail -1)"; }
for tool in memcheck racecheck synccheck; do
  S $tool tc python scripts/sanitize.py tc
  S $tool tcv python scripts/sanitize.py tcv
  S $tool ws python scripts/sanitize.py ws
  S $tool fb python scripts/sanitize.py fb
  S $tool codes python -m pytest -x -q -p no:cacheprovider "tests/test_gpu_codes.py::test_code_search_bit_exact[64-1000-HIGH]" "tests/test_gpu_codes.py::test_search_v3_parity[3-1-0.01-100-64-2-1]"
  S $tool idc python -m pytest -x -q -p no:cacheprovider "tests/test_gpu_idlist.py::test_search_idc_parity[3-1-64-3-1-500-HIGH]"
  S $tool scored python -m pytest -x -q -p no:cacheprovider "tests/test_gpu_scorers.py::test_search_scored_parity[hadamard-3-64-3-100-ALL-kw1]" "tests/test_gpu_scorers.py::test_search_scored_parity[mol-1-64-4-50-HIGH4-kw4]"
done
ls $O
