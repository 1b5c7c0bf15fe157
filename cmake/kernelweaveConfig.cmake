# CMake package for the B200 build of kernelweave: the drop-in for the reference's exported
# target (core/CMakeLists.txt: install(EXPORT …) → kernelweave::core). Downstream projects keep
#   find_package(kernelweave REQUIRED)
#   target_link_libraries(app PRIVATE kernelweave::core)
# and point CMAKE_PREFIX_PATH (or kernelweave_DIR) at this directory.
get_filename_component(_kw_root "${CMAKE_CURRENT_LIST_DIR}/.." ABSOLUTE)
set(_kw_lib "${_kw_root}/paper_1602_08477_b200/libkw_b200.so")
if(NOT EXISTS "${_kw_lib}")
  set(kernelweave_FOUND FALSE)
  set(kernelweave_NOT_FOUND_MESSAGE "libkw_b200.so not built: run __graft_entry__.build()")
  return()
endif()
if(NOT TARGET kernelweave::core)
  add_library(kernelweave::core SHARED IMPORTED)
  set_target_properties(kernelweave::core PROPERTIES
    IMPORTED_LOCATION "${_kw_lib}"
    INTERFACE_INCLUDE_DIRECTORIES "${_kw_root}/include"
    INTERFACE_COMPILE_FEATURES cxx_std_20)
endif()
set(kernelweave_FOUND TRUE)
set(kernelweave_VERSION 0.1)
