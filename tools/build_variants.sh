# parallel tuning builds: bash tools/build_variants.sh "name1:-DA=1 -DB=2" "name2:..."
for spec in "$@"; do
  name=${spec%%:*}; defs=${spec#*:}
  python tools/build_variant.py $name $defs > /tmp/bv_$name.log 2>&1 &
done
wait
for spec in "$@"; do name=${spec%%:*}; tail -1 /tmp/bv_$name.log; done
