# Developer A/B driver (GPU box): variants of the interface-iteration kernel
set -u
run() { echo "== $1"; BX_LIB=$2 python tools/sweep_part.py child 2 4096 8192; BX_LIB=$2 python tools/sweep_part.py child 1 8192 8192; }
run base paper_1804_09666_b200/libbandix_b200.so
for v in "$@"; do
  d=/tmp/v_$(echo "$v" | tr -c 'A-Za-z0-9' '_')
  python tools/variant_lib.py $d $v > /dev/null 2>&1; run "$v" $d/libbandix_b200.so
done
