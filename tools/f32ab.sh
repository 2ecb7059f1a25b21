cd "${GRAFT_REPO_ROOT:-/root/repo}"
for v in main f5 f6; do
  if [ "$v" = main ]; then unset STENCIL_B200_LIB; else export STENCIL_B200_LIB=tunelibs/lib_$v.so; fi
  echo "== $v"; timeout 300 python tools/f32_3d.py 2>&1 | grep box
done
