#!/bin/bash
# experimental build of the package with extra defines: tools/expbuild.sh <name> "-DFOO -DBAR"
# (expbuild/<name>/ holds a copy of the package + include; delete it after use: it travels with gpurun)
set -e
cd "$(dirname "$0")/.."
rm -rf expbuild/$1 && mkdir -p expbuild/$1
cp -r include expbuild/$1/
cp -r paper_1904_06971_b200 expbuild/$1/ && rm -f expbuild/$1/paper_1904_06971_b200/*.so && rm -rf expbuild/$1/paper_1904_06971_b200/__pycache__
cd expbuild/$1/paper_1904_06971_b200/csrc
make -j16 NVFLAGS="-std=c++17 --expt-relaxed-constexpr -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -Xcompiler -fPIC -DSG_MAX_P=4 -Xptxas -warn-spills $2" BUILD=../../build/csrc > ../../build.log 2>&1 || { tail -20 ../../build.log; exit 1; }
rm -rf ../../build
echo "built expbuild/$1"
