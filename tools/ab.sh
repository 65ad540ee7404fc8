# A/B of library builds: bash tools/ab.sh name1 name2 ... (variants/libsdv2_<name>.so; "main" = in-tree)
mkdir -p gpurun_out
for rep in 1 2; do
for v in "$@"; do
  if [ "$v" = main ]; then lib=""; else lib="--lib $PWD/paper_2511_07399_b200/variants/libsdv2_$v.so"; fi
  r=$(timeout 300 python bench.py --no-cpu-baseline --steps 100 $lib 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['ms_per_step'],3), {k: round(v['ms_per_step'],3) for k,v in d['roofline']['classes'].items()})")
  echo "$v: $r"
done
done
