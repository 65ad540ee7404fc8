# attention kernel time per library build: bash tools/time_attn_ab.sh name... (variants/libsdv2_<name>.so, main)
for v in "$@"; do
  if [ "$v" = main ]; then unset SDV2_LIB_PATH; else export SDV2_LIB_PATH=$PWD/paper_2511_07399_b200/variants/libsdv2_$v.so; fi
  echo "== $v"; timeout 90 python tools/time_attn.py | head -2
done
unset SDV2_LIB_PATH
