# build a variant of libmrep.so with extra nvcc defines: build_variant.sh NAME "-DFOO=1 ..."
# (A/B experiments: MREP_LIB=build/variants/libmrep_NAME.so python bench.py ...)
set -e
name=$1; shift
mkdir -p build/variants
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false -std=c++17 -Xcompiler -fPIC -Xcompiler -ffp-contract=off -Xcompiler -fvisibility=hidden -I include"
/usr/local/cuda/bin/nvcc $F $* -c paper_2504_11498_b200/csrc/mrep_project.cu -o build/variants/project_$name.o
objs=$(ls build/*.o | grep -v mrep_project.o)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build/variants/libmrep_$name.so $objs build/variants/project_$name.o -lcudart_static -lrt -lpthread -ldl
