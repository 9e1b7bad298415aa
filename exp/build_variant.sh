# build_variant.sh OUT.so [nvcc -D flags...]: the engine library with extra defines
set -e
out=$1; shift
d=$(mktemp -d)
cd /root/repo/paper_2506_23775_b200/csrc
for s in gf_ops gf_engine gf_target; do nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -cudart static "$@" -c -o $d/$s.o $s.cu 2>/dev/null & done; wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o /root/repo/$out $d/*.o
rm -rf $d
