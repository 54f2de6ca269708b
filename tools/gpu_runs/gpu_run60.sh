make -B > /dev/null 2>&1 || exit 1
timeout 600 python -c "import __graft_entry__ as g; g.build(); g.smoke()"
