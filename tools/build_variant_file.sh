# build variants/libdg_<name>.so from one csrc file with a sed expression applied (A/B experiments)
# usage: tools/build_variant_file.sh FILE.cu NAME 'sed-expr'
set -e
file=$1; name=$2; expr=$3
cd /root/repo
python -m paper_1907_08492_b200.build > /dev/null
mkdir -p variants /tmp/variant_$name
src=paper_1907_08492_b200/csrc/$file
tmp=/tmp/variant_$name/variant_tmp_${name}.cu   # outside csrc/ so that concurrent main builds never see it
sed "$expr" $src > $tmp
cmp -s $src $tmp && { echo "sed changed nothing"; rm $tmp; exit 1; }
inc=$(python -c "import sys; sys.path.insert(0,'paper_1907_08492_b200'); import build; print(build._nccl_dirs()[0])")
lib=$(python -c "import sys; sys.path.insert(0,'paper_1907_08492_b200'); import build; print(build._nccl_dirs()[1])")
nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr -O3 -std=c++17 \
  -I$inc -Iinclude -Ipaper_1907_08492_b200/csrc -c $tmp -o /tmp/variant_$name/$file.o
rm $tmp
objs=$(ls build/dg_b200/*.o | grep -v "/$file.o")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o variants/libdg_$name.so $objs /tmp/variant_$name/$file.o -L$lib -lnccl -lcudart -lquadmath -Xlinker -rpath=$lib
echo variants/libdg_$name.so
