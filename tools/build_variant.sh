# usage: bash tools/build_variant.sh <name> "<extra nvcc flags>" ; builds lib/libevoattn_<name>.so (A/B variants)
set -e
python -c "
import sys; from paper_2310_04610_b200 import build as B
B.build(force=True, out=B.LIBDIR + '/libevoattn_$1.so', extra='$2'.split())"
