# Build tuning variants of libgnpc.so into var/<name>.so (usage: tools/variants.sh name "defs" ...)
set -e
cd "$(dirname "$0")/.."
while [ $# -ge 2 ]; do
  GNPC_NVCC_DEFS="$2" python -c "from paper_2406_00809_b200 import build; build.build_lib(force=True)" > /tmp/var_$1.log 2>&1 || { tail -20 /tmp/var_$1.log; exit 1; }
  cp paper_2406_00809_b200/libgnpc.so var/$1.so; echo "built var/$1.so ($2)"
  shift 2
done
python -c "from paper_2406_00809_b200 import build; build.build_lib(force=True)" > /tmp/var_default.log 2>&1
