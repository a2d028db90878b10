# Build a variant libgdi.so into abtest/NAME with extra nvcc defines (same-box A/B:
# LD_LIBRARY_PATH=abtest/NAME picks it up ahead of the in-tree lib through RUNPATH).
#   bash scripts/build_ab.sh NAME "-DFOO=1 -DBAR"
NAME=$1; DEFS=$2
make -j8 BUILD=abtest/$NAME/build LIBDIR=abtest/$NAME NVCC="nvcc $DEFS" abtest/$NAME/libgdi.so > abtest/$NAME.buildlog 2>&1 || { tail -20 abtest/$NAME.buildlog; exit 1; }
echo "built abtest/$NAME/libgdi.so ($DEFS)"
