mkdir -p gpurun_out
for lib in paper_2505_21319_b200/lib/libefunc.so paper_2505_21319_b200/lib/variants/*/libefunc.so; do
  echo "$lib"; EFUNC_LIB_PATH=$PWD/$lib timeout 300 python tools/table4.py 2>/dev/null | grep -E "^\| (16|32)\^3 \| inf"
done
