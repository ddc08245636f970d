#!/bin/bash
# Builds an A/B variant of the library: paper_2505_24179_b200/lib_alt/libsale_b200_<name>.so
# from the current sources with csrc/<file> replaced by <replacement>.
#   tools/build_alt.sh <name> <replacement.cu> [<file in csrc>]   (default file: attention.cu)
# Selected at run time with SALE_B200_LIB=.../lib_alt/libsale_b200_<name>.so.
set -e
name=$1; repl=$2; file=${3:-attention.cu}
root=$(cd "$(dirname "$0")/.." && pwd)
pkg=$root/paper_2505_24179_b200
src=$pkg/build_alt/src_$name
rm -rf "$src"; mkdir -p "$src/csrc" "$pkg/lib_alt"
cp "$pkg"/csrc/* "$src/csrc/"
cp "$repl" "$src/csrc/$file"
sed -e 's#-I../include#-I'"$root"'/include#' "$pkg/Makefile" > "$src/Makefile"
sed -i -e 's#\.\./include/sale_b200.h#'"$root"'/include/sale_b200.h#g' "$src/Makefile"
make -s -j16 -C "$src" lib/libsale_b200.so
cp "$src/lib/libsale_b200.so" "$pkg/lib_alt/libsale_b200_$name.so"
echo "built $pkg/lib_alt/libsale_b200_$name.so"
