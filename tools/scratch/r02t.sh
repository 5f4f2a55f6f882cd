python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo BUILD FAILED; exit 1; }
for c in larger stress; do DI_DEBUG_MC=1 python tools/time_stages.py $c 20 2>&1 | tail -2; done
for c in larger; do DI_EXP_NO_MC=1 python tools/time_stages.py $c 20 2>&1 | tail -1; done
