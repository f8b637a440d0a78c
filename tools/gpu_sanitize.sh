# compute-sanitizer over tools/sanitize.py: memcheck / synccheck / initcheck on the product library,
# racecheck on build/liblsk_san.so (every thread arrives on the row-sum mbarriers; tools/build_sanitize.sh)
mkdir -p gpurun_out
for tool in memcheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize.py > gpurun_out/san_$tool.log 2>&1; echo "$tool rc $? $(grep 'SUMMARY' gpurun_out/san_$tool.log)"
done
LSK_LIB=build/liblsk_san.so timeout 900 compute-sanitizer --tool racecheck --print-limit 30 python tools/sanitize.py > gpurun_out/san_racecheck.log 2>&1; echo "racecheck rc $? $(grep 'SUMMARY' gpurun_out/san_racecheck.log)"
