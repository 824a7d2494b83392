#!/bin/bash
# tools/ab_variant.sh NAME -- snapshot the current in-tree library as
# tools/_bin/NAME/libmlnmf_b200.so (git-ignored; travels with gpurun) so two
# kernel variants can be timed alternately on the same box:
#   MLNMF_B200_LIB=tools/_bin/NAME/libmlnmf_b200.so python tools/profile_products.py ...
set -e
mkdir -p "tools/_bin/$1"
cp paper_1009_0881_b200/_lib/libmlnmf_b200.so "tools/_bin/$1/"
echo "tools/_bin/$1/libmlnmf_b200.so"
