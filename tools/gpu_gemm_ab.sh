# standalone GEMM times of prebuilt library variants (tools/_ab/lib_<tag>.so): $@ = tags
for rep in 1 2; do
  for v in "$@"; do
    cp tools/_ab/lib_$v.so paper_2603_09237_b200/libmorlax_b200.so
    echo "== $v $(timeout 120 python tools/gemm_time.py 2>&1 | tail -1)"
  done
done
