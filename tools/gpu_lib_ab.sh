# Same-session A/B of K1 library variants (tools/build_variant.sh): pass time + result checksum.
mkdir -p gpurun_out
V=${VARIANTS:-fastdiv}
args="DS_NONE=0"
for v in $V; do args="$args DAGSCHED_LIB=build/$v/libdagsched_b200.so"; done
args="$args DS_NONE=1"
for v in $V; do args="$args DAGSCHED_LIB=build/$v/libdagsched_b200.so"; done
timeout 900 python tools/k1_env_ab.py $args > gpurun_out/lib_ab.log 2>&1; echo "ab rc $?"
cat gpurun_out/lib_ab.log
