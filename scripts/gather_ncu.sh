# ncu sector counts of the guess kernel for several builds (each copied over the in-tree lib)
cd $GRAFT_REPO_ROOT
cp paper_2604_22312_b200/libgvrtopk.so /tmp/lib_keep.so
for l in "$@"; do
  cp $l paper_2604_22312_b200/libgvrtopk.so
  echo "== $l"
  timeout 300 ncu --metrics lts__t_sectors_srcunit_tex_op_read.sum,dram__bytes_read.sum,gpu__time_duration.sum -k regex:gvr_guess_kernel -s 2 -c 1 python scripts/prof_kernels.py 2>&1 | grep -E "lts__|dram__|gpu__time"
done
cp /tmp/lib_keep.so paper_2604_22312_b200/libgvrtopk.so
