#!/usr/bin/env bash
# Build A/B variants of libgbg.so that differ only in one source file's
# -D flags: profiles/mkvar.sh <file.cu> name1 "<flags1>" [name2 "<flags2>" ...]
# -> profiles/ab/<name>.so (other objects from paper_2405_11671_b200/_build)
set -eu
cd "$(dirname "$0")/.."
SRC=$1; shift
PKG=paper_2405_11671_b200
python -m $PKG.build > /dev/null
mkdir -p profiles/ab /tmp/gbgvar
OTHERS=$(ls $PKG/_build/*.o | grep -v "/${SRC%.cu}.o$")
while [ $# -gt 0 ]; do
  name=$1; flags=$2; shift 2
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --extended-lambda \
    -Xcompiler -fPIC -Xcompiler -O2 -Xptxas -O3 -DNDEBUG $flags -c $PKG/csrc/$SRC -o /tmp/gbgvar/$name.o
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o profiles/ab/$name.so /tmp/gbgvar/$name.o $OTHERS -lcudart
  echo "built profiles/ab/$name.so ($flags)"
done
