# build variants/libdg_<name>.so from k_kron4.cu with a sed expression applied (A/B experiments)
# usage: tools/build_variant.sh NAME 'sed-expr'
set -e
name=$1; expr=$2
cd /root/repo
python -m paper_1907_08492_b200.build > /dev/null
mkdir -p variants /tmp/variant_$name
sed "$expr" paper_1907_08492_b200/csrc/k_kron4.cu > paper_1907_08492_b200/csrc/k4_variant_tmp.cu
cmp -s paper_1907_08492_b200/csrc/k_kron4.cu paper_1907_08492_b200/csrc/k4_variant_tmp.cu && { echo "sed changed nothing"; rm paper_1907_08492_b200/csrc/k4_variant_tmp.cu; exit 1; }
inc=$(python -c "import sys; sys.path.insert(0,'paper_1907_08492_b200'); import build; print(build._nccl_dirs()[0])")
lib=$(python -c "import sys; sys.path.insert(0,'paper_1907_08492_b200'); import build; print(build._nccl_dirs()[1])")
nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr -O3 -std=c++17 \
  -I$inc -Iinclude -Ipaper_1907_08492_b200/csrc -c paper_1907_08492_b200/csrc/k4_variant_tmp.cu -o /tmp/variant_$name/k_kron4.o
rm paper_1907_08492_b200/csrc/k4_variant_tmp.cu
objs=$(ls build/dg_b200/*.o | grep -v k_kron4.cu.o)
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o variants/libdg_$name.so $objs /tmp/variant_$name/k_kron4.o -L$lib -lnccl -lcudart -lquadmath -Xlinker -rpath=$lib
echo variants/libdg_$name.so
