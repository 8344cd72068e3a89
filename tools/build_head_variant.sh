#!/bin/bash
# ab/lib_<name>.so = the in-tree build with <file> taken from git revision <rev>
# usage: tools/build_head_variant.sh <name> <rev> <csrc file>
set -e
name=$1; rev=$2; f=$3
mkdir -p ab/obj_$name
git show $rev:paper_2109_05948_b200/csrc/$f > ab/obj_$name/$f
objs=""
for o in paper_2109_05948_b200/build/*.o; do
  b=$(basename $o .o)
  if [ "$b.cu" = "$f" ]; then
    nvcc -ccbin /usr/bin/g++ -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 \
      --expt-relaxed-constexpr -I include -I paper_2109_05948_b200/csrc -c ab/obj_$name/$f -o ab/obj_$name/$b.o
    objs="$objs ab/obj_$name/$b.o"
  else
    objs="$objs $o"
  fi
done
nvcc -ccbin /usr/bin/g++ -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC -o ab/lib_$name.so $objs
echo ab/lib_$name.so
